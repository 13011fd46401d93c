"""Build libctrecon.so in-tree for sm_100a (nvcc, no fast-math)."""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libctrecon.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I" + os.path.join(HERE, "..", "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "ctrecon.h"),
                                                                 __file__]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force=False, verbose=False, extra=(), out=None):
    """Each .cu compiles to an object in parallel (no cross-file device code), then one link.
    out: another output path (tuning variants built with extra -D flags; not the product)."""
    lib = out or LIB
    if out is None and not force and up_to_date():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    tmpdir = os.path.join(HERE, ".build%d" % os.getpid())
    os.makedirs(tmpdir, exist_ok=True)
    objs = [os.path.join(tmpdir, os.path.basename(src)[:-3] + ".o") for src in sources()]
    cflags = [f for f in FLAGS if f != "-shared"]

    def compile_one(pair):
        src, obj = pair
        cmd = [NVCC] + cflags + list(extra) + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)

    try:
        with ThreadPoolExecutor(max_workers=min(8, len(objs))) as ex:
            list(ex.map(compile_one, zip(sources(), objs)))
        tmp = lib + ".tmp%d" % os.getpid()
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC"] + objs + \
              ["-o", tmp, "-lnccl", "-lcudart"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(tmp, lib)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
        os.rmdir(tmpdir)
    return lib


if __name__ == "__main__":
    build(force=True, verbose=True, extra=sys.argv[1:])
    print(LIB)
