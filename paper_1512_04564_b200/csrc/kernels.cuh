// kernels.cuh — host-side launcher declarations for libctrecon.so kernels.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "ct_internal.cuh"

namespace ctr {

// Programmatic dependent launch (PDL) for the kernels of a solver sub-iteration: while g_pdl is
// set (the single-GPU sub-iteration graph's capture), launch_k launches with programmatic stream
// serialization; every such kernel starts with pdl_enter(), which waits for its predecessor's
// completion and memory (griddepcontrol.wait) before touching any data.  The dependent grid is
// launched at the predecessor's exit (implicit trigger): c1 +2.2%, c2 +0.4% (launch latency).  An
// early trigger at kernel entry (griddepcontrol.launch_dependents, CTR_PDL_TRIGGER=1) let waiting
// blocks occupy the SMs during the predecessor's tail and was slower (c1 -26%, c3 -12%;
// profiles/r2s/pdl_ab.log).  Without the launch attribute both instructions are no-ops.
extern thread_local bool g_pdl;

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    if (!g_pdl) {
        kern<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#ifndef CTR_PDL_TRIGGER
#define CTR_PDL_TRIGGER 0   // 1: early trigger at kernel entry (measured: c1 -26%, c3 -12%)
#endif
__device__ __forceinline__ void pdl_enter() {
#if CTR_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

enum FwdMode { FWD_PLAIN = 0, FWD_RESID = 1, FWD_ONES_W = 2 };
enum BackEpi { BK_WRITE = 0, BK_ACCUM = 1, BK_INIT = 2, BK_UPDATE = 3 };

struct RegParams {
    float beta[13];
    float delta, inv_delta, delta2;   // delta2 = delta^2 (UPD_RAW hyperbola)
    int potential, n_dirs;
    int maxcurv;          // D_R with omega(0) = 1 (CT_CURV_MAX)
    float bsum;           // sum_d 2 beta_d: the interior maximum-curvature sum
    float q, qexp;        // q-GGMRF exponent q and 2 - q
};

// x_pair: (xa, xb); with ctl != nullptr the forward reads the buffer written
// by this sub-iteration's update (parity of k - k_base), else xa.
void launch_fwd(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, int max_count, const float* xa,
                const float* xb, const float* y, const float* w, float* out, int mode, cudaStream_t s,
                int pfx_stride = 0);  // > 0: xa is the float2 z-prefix array (3-D solve path)

// Segmented z-prefix forward (volumes whose z-prefix exceeds L2): nseg segments of
// seg_len slabs along each wedge; sched from fwd_seg_schedule (device copy, nsched entries); part =
// nseg * max_count * nt * ns floats of raw segment sums, reduced in segment order into out with the
// forward's epilogue (mode as launch_fwd).
int fwd_seg_len(const DGeom& G, int nseg);
std::vector<int2> fwd_seg_schedule(const DGeom& G, const std::vector<float4>& htab, Views v, int count, int nseg,
                                   int* seg_len);
void launch_fwd_seg(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, int max_count, const float* pfx,
                    const float* y, const float* w, float* out, int mode, cudaStream_t s, int pfx_stride,
                    const int2* sched, int nsched, int seg_len, int nseg, float* part);

// z-prefix array of x+ for the 3-D forward (written by the update kernel):
// per voxel column, float2 Q_k = (A_k, x_k) for k = 0..nz-1 and Q_nz = (P_nz, 0),
// P_k = sum_{k'<k} x_k', A_k = P_k - (k - 1/2) x_k (the cumulative at voxel coordinate
// f in [k - 1/2, k + 1/2] is A_k + f x_k).  Column stride in float2 units: nz + 1 rounded up to even.
__host__ __device__ inline int pfx_stride_of(const DGeom& G) { return ((G.nz + 1) + 1) & ~1; }

// z-prefix array of x (same entries as the update kernel writes for x+), for ct_forward_zprefix
void launch_zprefix(const DGeom& G, const float* x, float* pfx, cudaStream_t s);
// r_out = r / L_z(s, t) over `count` views (the solver's residual buffer carries L_z for the back-projector)
void launch_unfold_lz(const DGeom& G, int count, const float* r, float* r_out, cudaStream_t s);

void launch_back(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* proj, float scale,
                 int epi, bool apply_lz, float* out, float* g, float* ht, cudaStream_t s);

// regulariser gradient / curvature only (ct_reg_grad)
// (halo_lo / halo_hi: planes -1 / nz of x exist, G a z-slab of a larger volume)
void launch_reg(const DGeom& G, const RegParams& rp, const float* x, const float* kappa, float* grad, float* curv,
                cudaStream_t s, bool halo_lo = false, bool halo_hi = false);

// fused stencil + x-update of Algorithm 1 lines 4-5, writes htilde partial
void launch_update(const DGeom& G, const RegParams& rp, const Ctl* ctl, float* xa, float* xb, const float* dl,
                   const float* g, float* ht, const float* kappa, float box_lo, float box_hi, float* pfx,
                   cudaStream_t s);

// z-slab decomposition: the update with one halo plane of x below / above the slab
// (x buffers xa, xb point at plane 0 of (nz + 2)-plane allocations)
void launch_update_halo(const DGeom& G, const RegParams& rp, const Ctl* ctl, float* xa, float* xb, const float* dl,
                        float* g, float* ht, float box_lo, float box_hi, float* pfx, bool halo_lo, bool halo_hi,
                        cudaStream_t s, const float* kappa = nullptr);

// multi-GPU path: fold the all-reduced zeta of the previous sub-iteration into
// g, htilde (lines 7-8) and run lines 4-5 from precomputed grad R / D_R
// (launch_reg on the new x); Ctl.k is one behind (the advance follows)
void launch_update_pre(const DGeom& G, const Ctl* ctl, const float* xin, float* xout, const float* dl, float* g,
                       float* ht, const float* zeta, const float* grad, const float* curv, float box_lo,
                       float box_hi, float* pfx, cudaStream_t s);

// FBP / FDK initialiser (fbp.cu): filtered sinogram into qbuf (na views), image into out
void launch_fbp(const DGeom& G, const float4* vtab, const float* proj, float* qbuf, float* out, double dsd,
                cudaStream_t s);

// elementwise helpers of ct_kappa_weights: fill with a constant; kappa = sqrt(a / b), 0/0 = 1
void launch_fill(float* p, long long n, float v, cudaStream_t s);
void launch_kappa_ratio(long long n, const float* a, const float* b, float* kappa, cudaStream_t s);

// dist path: g, htilde update from an all-reduced zeta (lines 7-8)
void launch_gh_update(const DGeom& G, const Ctl* ctl, const float* zeta, float* g, float* ht, cudaStream_t s);
void launch_init_from_zeta(const DGeom& G, const float* zeta, float* g, float* ht, cudaStream_t s);
void launch_advance(Ctl* ctl, cudaStream_t s, int n = 1);   // k += 1 in n consecutive control blocks
// base[i] = sum_p base[p stride + i], p = 0..n-1 in order (emulated reduction of partial gradients)
void launch_sum_partials(float* base, int n, long long stride, long long count, cudaStream_t s);
void launch_state_h(const DGeom& G, const float* dl, const float* x, const float* ht, float* h, cudaStream_t s);
// flag[0] |= any non-finite in x; optional sum of squares of (x - xref) into dsum[0]
void launch_check(const DGeom& G, const float* x, const float* xref, int* flag, double* dsum, cudaStream_t s);

// nonzero entries of A on views v, added into *count (device)
void launch_count(const DGeom& G, const float4* vtab, Views v, unsigned long long* count, cudaStream_t s);
// count3[0] += nnz, count3[1] += in-cone voxel-view pairs, count3[2] += in-cone column-view pairs
void launch_count_work(const DGeom& G, const float4* vtab, Views v, unsigned long long* count3, cudaStream_t s);

int64_t launches_add(int64_t n);  // launch accounting

}  // namespace ctr
