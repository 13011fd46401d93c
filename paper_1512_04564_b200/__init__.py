"""B200-native hot path of relaxed OS-LALM for PWLS CT (arXiv 1512.04564).

    ctrecon   thin ctypes binding of libctrecon.so (include/ctrecon.h)
    recon     device-tensor setup around the C-ABI (no method arithmetic)
    csrc/     sm_100a CUDA kernels + the C-ABI implementation

The CUDA library is the only compute path: importing `ctrecon` functions
raises if libctrecon.so is missing; there is no CPU fallback.
"""
