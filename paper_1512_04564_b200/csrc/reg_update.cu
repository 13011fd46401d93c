// reg_update.cu — K4 regulariser stencil (Eq. 35) and the
// fused Algorithm 1 x-update (lines 4-5), the multi-GPU
// fold-and-update kernel, plus the small elementwise kernels of the solver
// (dist-path g/htilde update, advance of the Eq. 37 counter, htilde -> h,
// finiteness / RMS check).
//
// grad_j = sum_n beta_{d(j,n)} kappa_j kappa_n phi'(x_j - x_n)
// D_R,j  = 2 sum_n beta_{d(j,n)} kappa_j kappa_n omega(x_j - x_n),  omega = phi'(t)/t
// over the in-volume neighbours n (26 in 3-D, 8 in 2-D).
//
// Update (htilde = D_L x - h):
//   s   = rho htilde + (1 - rho) g
//   x+  = clamp(x - (s + grad)/(rho D_L + D_R), box)   (denominator 0 keeps x)
//   htilde_partial = (1 - alpha) (D_L (x+ - x) + htilde)   (completed by the
//                     back-projection epilogue: htilde+ = htilde_partial + alpha zeta)
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace ctr {

// compile-time direction offsets for the register-window stencil (fold after unrolling)
__host__ __device__ constexpr int dir_x(int d) {
    return (d == 0 || d == 2 || d == 3 || d == 5 || d == 9 || d == 11) ? 1 : (d == 6 || d == 10 || d == 12) ? -1 : 0;
}
__host__ __device__ constexpr int dir_y(int d) {
    return (d == 1 || d == 2 || d == 7 || d == 9 || d == 10) ? 1 : (d == 3 || d == 8 || d == 11 || d == 12) ? -1 : 0;
}
__host__ __device__ constexpr int dir_z(int d) { return d >= 4 ? 1 : 0; }

static_assert(dir_x(6) == -1 && dir_y(8) == -1 && dir_z(4) == 1 && dir_x(4) == 0 && dir_y(12) == -1 &&
                  dir_x(11) == 1 && dir_y(11) == -1 && dir_z(3) == 0,
              "direction table");

// UPD_RAW (hyperbola only): the register window holds x itself, not x/delta, and omega is
// evaluated as o' = 1/sqrt(delta^2 + t^2) = omega/delta, so that t o' = tp omega (the gradient
// sum is unchanged) and the curvature sum is delta sum w o' -- no per-plane scaling of the window.
// Measured slower (c4 update 0.356 vs 0.339 ms, c3 0.077 vs 0.071; profiles/r2z/raw_ab.log): kept
// as a switch only
#ifndef UPD_RAW
#define UPD_RAW 0
#endif
template <int POT>
__host__ __device__ constexpr bool upd_raw() { return UPD_RAW && POT == 1; }

// Potential in scaled form: tp = t / delta.  Returns omega(t) = phi'(t)/t and
// tp * omega; phi'(t) = delta * tp * omega for all three potentials.
template <int POT>
__device__ __forceinline__ float omega_scaled(float tp, const RegParams& rp) {
    if (POT == 0) return 1.f;                                   // quadratic
    if (POT == 1) return rsqrt_ftz(fmaf(tp, tp, 1.f));          // hyperbola
    if (POT == 2) return __fdividef(1.f, 1.f + fabsf(tp));      // Fair
    // q-GGMRF (p = 2): u = |t/delta|^(2-q), omega = (2 + q u) / (2 (1 + u)^2)
    const float u = exp2f(rp.qexp * __log2f(fmaxf(fabsf(tp), 1e-30f)));   // 0^0 = 1 when q = 2
    const float v = 1.f + u;
    return __fdividef(fmaf(rp.q, u, 2.f), 2.f * v * v);
}

// 26/8-neighbour sums over a register window W[slot][dy+1][dx+1] of x/delta
// whose planes z-1, z, z+1 sit in ring slots ZA, ZB, ZC (compile-time, so the
// z-march rotates slots instead of moving registers).  Returns
// gs = sum_n w_n tp_n omega_n and cs = sum_n w_n omega_n (w_n = beta kappa_j
// kappa_n); grad = delta gs, curv = 2 cs.  CHECK = false is the interior path:
// every neighbour exists, no predicates, and without kappa the two
// neighbours of a direction share one beta multiply.
// PATH: 0 interior (every neighbour exists), 1 checked (any border), 2 x-border only (every y and z
// neighbour exists): the interior arithmetic with the differences to the missing x neighbours
// selected to 0 (their gradient term vanishes) and their curvature terms, beta_d omega(0) = beta_d
// each, subtracted afterwards (xcorr = (!im + !ip) sum_{d: ox != 0} beta_d, per column).
template <int NDIRS, bool KAPPA, int POT, int ZA, int ZB, int ZC, int PATH>
__device__ __forceinline__ void window_stencil(const float (&W)[4][3][3], const float (&K)[4][3][3],
                                               const RegParams& rp, bool im, bool ip, bool jm, bool jp, bool km,
                                               bool kp, float xcorr, float& gs_out, float& cs_out) {
    constexpr bool CHECK = PATH == 1;
    const float xv = W[ZB][1][1];
    const float kj = KAPPA ? K[ZB][1][1] : 1.f;
    float gs = 0.f, cs = 0.f, cmax = 0.f;
    // interior path: the two neighbours of a direction as one packed pair (FFMA2 / FMUL2), the
    // sums kept per half and added at the end
    float2 gs2 = make_float2(0.f, 0.f), cs2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int d = 0; d < NDIRS; d++) {
        const int ox = dir_x(d), oy = dir_y(d), oz = dir_z(d);
        const int zp = oz > 0 ? ZC : ZB, zm = oz > 0 ? ZA : ZB;
        if (!CHECK && !KAPPA) {
            float2 t = make_float2(xv - W[zp][1 + oy][1 + ox], xv - W[zm][1 - oy][1 - ox]);
            if (PATH == 2 && ox != 0) {
                t.x = (ox > 0 ? ip : im) ? t.x : 0.f;
                t.y = (ox > 0 ? im : ip) ? t.y : 0.f;
            }
            float2 o;
            if (POT == 1) {
                const float2 u = fma2(t, t, bcast2(upd_raw<POT>() ? rp.delta2 : 1.f));
#if UPD_DIAG & 8            // timing diagnostic only (wrong results): no MUFU in the interior stencil
                o = make_float2(u.x, u.y);
#else
                o = make_float2(rsqrt_ftz(u.x), rsqrt_ftz(u.y));
#endif
            } else {
                o = make_float2(omega_scaled<POT>(t.x, rp), omega_scaled<POT>(t.y, rp));
            }
            gs2 = fma2(bcast2(rp.beta[d]), mul2(t, o), gs2);
            cs2 = fma2(bcast2(rp.beta[d]), o, cs2);
        } else {
#pragma unroll
            for (int sg = 0; sg < 2; sg++) {
                const int sx = sg ? -ox : ox, sy = sg ? -oy : oy, sz = sg ? -oz : oz;
                const int zs = sg ? zm : zp;
                const bool ok = !CHECK || ((sx < 0 ? im : (sx > 0 ? ip : true)) &&
                                           (sy < 0 ? jm : (sy > 0 ? jp : true)) &&
                                           (sz < 0 ? km : (sz > 0 ? kp : true)));
                if (ok) {
                    const float wgt = KAPPA ? rp.beta[d] * kj * K[zs][1 + sy][1 + sx] : rp.beta[d];
                    const float t = xv - W[zs][1 + sy][1 + sx];
                    const float o = upd_raw<POT>() ? rsqrt_ftz(fmaf(t, t, rp.delta2)) : omega_scaled<POT>(t, rp);
                    gs = fmaf(wgt, t * o, gs);
                    cs = fmaf(wgt, o, cs);
                    cmax += wgt;
                }
            }
        }
    }
    if (!CHECK && !KAPPA) {
        gs = gs2.x + gs2.y;
        cs = cs2.x + cs2.y;
        if (upd_raw<POT>()) cs *= rp.delta;
        if (PATH == 2) cs -= xcorr;
    } else if (upd_raw<POT>()) {
        cs *= rp.delta;
    }
    gs_out = gs;
    // maximum curvature: omega(0) = 1 for every in-volume neighbour (interior, no kappa: bsum)
    cs_out = rp.maxcurv ? ((!CHECK && !KAPPA) ? (PATH == 2 ? rp.bsum - xcorr : rp.bsum) : cmax) : cs;
}

// Arguments of the update-family kernels (k_update, k_update_pre).
struct UpdArgs {
    float* xa;            // solver x double buffer (parity from Ctl unless xin is set)
    float* xb;
    const float* xin;     // UPD_STEN: explicit input image
    const float* dl;      // D_L
    float* g;             // g (k_update_pre folds the pending zeta into it)
    float* ht;            // htilde
    const float* kappa;   // NULL = ones
    const float* zeta;    // k_update_pre: all-reduced zeta of the previous sub-iteration
    const float* grad;    // k_update_pre: grad R(x) from the stencil kernel
    const float* curv;    // k_update_pre: D_R(x)
    float* grad_out;      // UPD_STEN outputs
    float* curv_out;
    float* pfx;           // z-prefix of x+ for the 3-D forward (NULL = none)
    float box_lo, box_hi;
    int CZ;               // voxels per z-chunk
    int halo_lo, halo_hi; // z-slab decomposition: planes -1 / nz of x exist (neighbour slabs' halos)
};

enum UpdMode { UPD_FULL = 0, UPD_STEN = 1 };

// z-prefix of the block's x+ columns (x+ staged in shared memory xs[k][lane]),
// written column by column by the row's warps (UPD_PFXT; the older form scanned the
// chunk totals across the NZC chunks and had each thread write the entries of its
// chunk): (A_k, x_k) as float2 with A_k = P_k - (k - 1/2) x_k and
// P_k = sum_{k'<k} x_k' (z-fastest, column stride pfx_stride_of(G)), plus
// (P_nz, 0) from the last chunk: the cumulative at voxel coordinate f in
// [k - 1/2, k + 1/2] is then one FFMA, A_k + f x_k.
// Columns w, w + nw, ... of the 32 staged columns i0 .. i0 + 31 of row j (xs[k * 33 + column]):
// lane = plane within a group of 32, warp scan of the group plus the carry of the groups below,
// one contiguous 256 B store of 32 (A_k, x_k) entries.  Shared by write_prefix and k_zprefix, so
// that the fused update and ct_forward_zprefix / the multi-GPU path build bit-identical prefixes.
__device__ __forceinline__ void prefix_columns(const DGeom& G, float* __restrict__ pfx, const float* xs, int w, int nw,
                                               int lane, int i0, int j) {
    if (j >= G.ny) return;
    const size_t stride = (size_t)pfx_stride_of(G);
    for (int cl = w; cl < 32 && i0 + cl < G.nx; cl += nw) {
        float2* __restrict__ pc = reinterpret_cast<float2*>(pfx) + ((size_t)j * G.nx + (size_t)(i0 + cl)) * stride;
        float carry = 0.f;
        for (int kb = 0; kb < G.nz; kb += 32) {
            const int k = kb + lane;
            const float xk = k < G.nz ? xs[k * 33 + cl] : 0.f;
            float inc = xk;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const float t = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += t;
            }
            float ex = __shfl_up_sync(0xffffffffu, inc, 1);
            if (lane == 0) ex = 0.f;
            const float P = carry + ex;
            if (k < G.nz) pc[k] = make_float2(fmaf(0.5f - (float)k, xk, P), xk);  // (A_k, x_k), one rounding
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) pc[G.nz] = make_float2(carry, 0.f);  // (P_nz, 0)
    }
}

#ifndef UPD_PFXT
#define UPD_PFXT 1   // 1: transposed write (a warp writes 32 consecutive entries of one column: 256 B per store);
                     // 0: every thread writes its own column's chunk (32 separate 8-byte sectors per store)
#endif
__device__ __forceinline__ void write_prefix(const DGeom& G, float* __restrict__ pfx, const float* xs, float* tot,
                                             float run, int c, int lane, bool act, unsigned col, int k0, int k1) {
    CTR_CHECK(c < (int)blockDim.y && k1 <= G.nz, "update prefix chunk");
#if UPD_PFXT
    // the row's NZC chunk-warps have staged x+ of the row's 32 columns (xs[k][lane]); after a named
    // barrier over them, warp c takes columns c, c + NZC, ...: lane = plane within a group of 32,
    // a warp scan gives P_k, and the 32 entries of the group go out as one contiguous 256 B store
    // (the per-thread form wrote 32 separate sectors per store and cost 27% of the kernel,
    // profiles/r2fh/update_diag.log)
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.z), "r"(32 * (int)blockDim.y) : "memory");
    prefix_columns(G, pfx, xs, c, (int)blockDim.y, lane, (int)blockIdx.x * 32, (int)(blockIdx.y * blockDim.z + threadIdx.z));
#else
    tot[c * 32 + lane] = run;
    // only the NZC chunk-warps of this row exchange totals (xs is per thread): a named
    // barrier per row instead of the whole block
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.z), "r"(32 * (int)blockDim.y) : "memory");
    float P = 0.f;
    for (int q = 0; q < c; q++) P += tot[q * 32 + lane];
    if (!act) return;
    float2* __restrict__ pc = reinterpret_cast<float2*>(pfx) + (size_t)col * (size_t)pfx_stride_of(G);
    for (int k = k0; k < k1; k++) {
        const float xk = xs[k * 33 + lane];
        pc[k] = make_float2(fmaf(0.5f - (float)k, xk, P), xk);  // (A_k, x_k), one rounding
        P += xk;
    }
    if (k1 == G.nz) pc[G.nz] = make_float2(P, 0.f);  // (P_nz, 0)
#endif
}

// Stencil (+ x-update).  Block = 32 consecutive i (a warp) x NZC z-chunks x
// JPB rows j; thread = one voxel column (i, j) over the z-chunk
// [c CZ, (c+1) CZ).  The 3x3 neighbourhood of x/delta (and kappa) of four
// planes lives in a register ring: plane k+2 and D_L, g, htilde of voxel k+1
// are fetched at the top of step k and first touched one step later (a full
// stencil of latency hiding); the march is unrolled by 4 so the ring slots are
// compile-time.  Interior planes of warps without an edge column take the
// predicate-free stencil (a warp-uniform choice: an edge warp runs the checked
// stencil on all its lanes instead of both paths); the JPB rows of a block share their
// x rows in L1.  32-bit element offsets (nvox < 2^32, ct_geom_create).
//   UPD_FULL (Algorithm 1 lines 4-5, the solve path): x+ and htilde_partial in
//     the boundary layout (coalesced over i); with pfx the z-prefix of x+.
//   UPD_STEN (ct_reg_grad, and the multi-GPU path where the stencil of the new
//     x overlaps the zeta all-reduce): grad R(x) and D_R(x) only.
#ifndef UPD_ZDIV
#define UPD_ZDIV 24
#endif
#ifndef UPD_CPA
#define UPD_CPA 0   // D_L, g, htilde through a cp.async shared-memory ring 3 voxels ahead (FULL mode);
                    // measured no faster (c4 0.341 vs 0.339 ms, profiles/r2z/cpa_ab.log): a switch only
#endif
#ifndef UPD_DIAG
#define UPD_DIAG 0   // timing diagnostics (results wrong; never the product build), bit mask: 1 no stencil arithmetic,
                     // 2 no z-prefix write, 4 no D_L / g / htilde loads, 8 no MUFU (profiles/r2fh/update_diag.log)
#endif
#ifndef UPD_MINB
#define UPD_MINB 3  // <= 80 registers: 3 blocks of 256 per SM
#endif
template <int POT, int NDIRS, bool KAPPA, int MODE>
__global__ void __launch_bounds__(256, UPD_MINB) k_update(DGeom G, RegParams rp, const Ctl* __restrict__ ctl, UpdArgs A) {
    pdl_enter();
    extern __shared__ float upd_sm[];  // pfx: xs[JPB][nz][33], tot[JPB][NZC][32]
    constexpr bool FULL = (MODE == UPD_FULL);
    const int lane = threadIdx.x, c = threadIdx.y, jj = threadIdx.z;
    const int NZC = blockDim.y;
    const int i = blockIdx.x * 32 + lane;
    const int j = blockIdx.y * blockDim.z + jj;
    const bool act = i < G.nx && j < G.ny;
    const float* __restrict__ x = A.xin;
    float* __restrict__ xn = nullptr;
    float rho = 0.f, alpha = 0.f;
    if (FULL) {
        const bool odd = ((ctl->k - ctl->k_base) & 1) != 0;
        x = odd ? A.xb : A.xa;
        xn = odd ? A.xa : A.xb;
        rho = rho_of_k(ctl);
        alpha = ctl->alpha;
    }
    const bool simple = FULL && ctl->simple;  // Algorithm 2: htilde holds zeta, not updated here
    const float idel = rp.inv_delta, del = rp.delta;
    const bool im = i > 0, ip = i + 1 < G.nx, jm = j > 0, jp = j + 1 < G.ny;
    const bool inxy = act && im && ip && jm && jp;
    const bool wfast = __all_sync(0xffffffffu, !act || inxy);   // warp-uniform stencil path (no divergence)
    const bool wxedge = !KAPPA && __all_sync(0xffffffffu, !act || (jm && jp));   // x-border only: PATH 2
    float xcorr = 0.f;
#pragma unroll
    for (int d = 0; d < NDIRS; d++)
        if (dir_x(d) != 0) xcorr += rp.beta[d];
    xcorr *= (float)(!im) + (float)(!ip);
    const unsigned nx = (unsigned)G.nx, nxy = (unsigned)G.nxy;
    const unsigned col = act ? (unsigned)j * nx + (unsigned)i : 0u;
    const int k0 = c * A.CZ, k1 = min(G.nz, k0 + A.CZ);
    float* xs = upd_sm + (size_t)jj * G.nz * 33;
    float* tot = upd_sm + (size_t)blockDim.z * G.nz * 33 + (size_t)(jj * NZC) * 32;
    const float* __restrict__ kappa = A.kappa;
    float W[4][3][3], K[4][3][3], XC[4];
    float Dv[2], Gv[2], Hv[2];  // D_L, g, htilde of the current / next voxel
    // raw loads into a ring slot; the slot is scaled by 1/delta one step later.
    // Interior columns load the 3x3 block unconditionally from a clamped plane (a
    // plane outside the volume is never weighted: the stencil checks km/kp there).
    const int klo = A.halo_lo ? -1 : 0, khi = A.halo_hi ? G.nz : G.nz - 1;   // readable planes of x
    const float* __restrict__ xlo = x + (long long)klo * (long long)nxy;       // plane klo (x and kappa)
    auto load_plane = [&](auto slot_c, int k) {
        constexpr int S = decltype(slot_c)::value;
        if (inxy) {
            // interior column: a 32-bit offset from the lowest readable plane klo (the halo plane
            // -1 of a z-slab lies below x); (kc - klo) * nxy + col - nx - 1 < 2^32
            const int kc = min(max(k, klo), khi);
            const unsigned off = (unsigned)(kc - klo) * nxy + col - nx - 1u;
            CTR_CHECK(col >= nx + 1u && (unsigned long long)(kc - klo) * nxy + col + nx + 1u <
                                            (unsigned long long)(khi - klo + 1) * nxy, "update window");
            const float* __restrict__ p = xlo + off;
            const float* __restrict__ pk = KAPPA ? kappa + (long long)klo * (long long)nxy + off : nullptr;
#pragma unroll
            for (int dy = 0; dy < 3; dy++) {
#pragma unroll
                for (int dx = 0; dx < 3; dx++) {
                    W[S][dy][dx] = __ldg(p + dx);
                    if (KAPPA) K[S][dy][dx] = __ldg(pk + dx);
                }

                p += nx;
                if (KAPPA) pk += nx;
            }
        } else {
            const bool ok = act && k >= klo && k <= khi;
            const long long o = ok ? (long long)k * nxy + col : 0;
#pragma unroll
            for (int dy = -1; dy <= 1; dy++) {
                const bool vy = dy < 0 ? jm : (dy > 0 ? jp : true);
                const long long ro = o + (long long)dy * (int)nx;
#pragma unroll
                for (int dx = -1; dx <= 1; dx++) {
                    const bool v = ok && vy && (dx < 0 ? im : (dx > 0 ? ip : true));
                    W[S][dy + 1][dx + 1] = v ? __ldg(x + (ro + dx)) : 0.f;
                    if (KAPPA) K[S][dy + 1][dx + 1] = v ? __ldg(kappa + (ro + dx)) : 0.f;
                }
            }
        }
    };
    auto scale_plane = [&](auto slot_c) {
        constexpr int S = decltype(slot_c)::value;
        XC[S] = W[S][1][1];
        const float sc = upd_raw<POT>() ? 1.f : idel;   // UPD_RAW: the window stays x (folded away)
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int b = 0; b < 3; b++) W[S][a][b] *= sc;
    };
    auto load_vox = [&](auto par_c, int k) {
        if (!FULL) return;
        constexpr int Q = decltype(par_c)::value;
        const unsigned idx = (unsigned)min(k, k1 - 1) * nxy + col;   // past the chunk: never used
        if (UPD_DIAG & 4) {   // timing diagnostic: no D_L / g / htilde loads
            Dv[Q] = Gv[Q] = Hv[Q] = (float)idx;
            return;
        }
        Dv[Q] = __ldg(A.dl + idx);
        Gv[Q] = __ldg(A.g + idx);
        Hv[Q] = A.ht[idx];
    };
    // UPD_CPA: D_L, g, htilde of voxel k + 3 are copied into a per-thread shared-memory ring slot
    // (k mod 4) by cp.async three steps ahead of their use (no registers held in flight)
    constexpr bool CPA = FULL && UPD_CPA;
    constexpr int nthr = 256;   // ring stride (>= threads per block)
    float* ring = upd_sm + (A.pfx ? (size_t)blockDim.z * G.nz * 33 + (size_t)blockDim.z * NZC * 32 : 0) +
                  ((jj * NZC + c) * 32 + lane);
    auto issue_vox = [&](int k) {
        if (!CPA) return;
        if (act && k < k1) {
            const unsigned idx = (unsigned)k * nxy + col;
            float* r = ring + ((k & 3) * 3) * nthr;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(r)),
                         "l"(__cvta_generic_to_global(A.dl + idx)) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(r + nthr)),
                         "l"(__cvta_generic_to_global(A.g + idx)) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(r + 2 * nthr)),
                         "l"(__cvta_generic_to_global(A.ht + idx)) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");   // one group per voxel, empty past the chunk
    };
    float run = 0.f;
    // voxel k: planes k-1, k, k+1 in slots ZA, ZB, ZC (ZC loaded raw one step
    // ago: scaled now); plane k+2 is fetched into ZD and D_L, g, htilde of
    // voxel k+1 into the other parity -- both are consumed one step later.
    auto step = [&](auto za, auto zb, auto zc, auto zd, int k) {
        constexpr int ZA = decltype(za)::value, ZB = decltype(zb)::value, ZC = decltype(zc)::value;
        constexpr int Q = ZB & 1;
        scale_plane(zc);
        load_plane(zd, k + 2);
        if (CPA) issue_vox(k + 3);
        else load_vox(std::integral_constant<int, Q ^ 1>(), k + 1);
        float xnew = 0.f;
        if (act) {
            const unsigned idx = (unsigned)k * nxy + col;
            float gs, cs;
            // (2-D: no z neighbours, so the z borders do not force the checked stencil)
            const bool km = NDIRS == 4 || k > 0 || A.halo_lo, kp = NDIRS == 4 || k + 1 < G.nz || A.halo_hi;
            if ((UPD_DIAG & 1) && wfast && km && kp) {   // timing diagnostic: no stencil arithmetic
                gs = W[ZA][0][0] + W[ZA][2][2] + W[ZC][0][2] + W[ZC][2][0] + W[ZB][1][0] + W[ZB][1][2] + W[ZB][0][1] +
                     W[ZB][2][1] + W[ZA][1][1];
                cs = W[ZC][1][1] + W[ZA][0][1] + W[ZA][0][2] + W[ZA][1][0] + W[ZA][1][2] + W[ZA][2][0] + W[ZA][2][1] +
                     W[ZB][0][0] + W[ZB][0][2] + W[ZB][2][0] + W[ZB][2][2] + W[ZC][0][0] + W[ZC][0][1] + W[ZC][1][0] +
                     W[ZC][1][2] + W[ZC][2][1] + W[ZC][2][2];
            } else if (wfast && km && kp)
                window_stencil<NDIRS, KAPPA, POT, ZA, ZB, ZC, 0>(W, K, rp, im, ip, jm, jp, km, kp, xcorr, gs, cs);
            else if (wxedge && km && kp)
                window_stencil<NDIRS, KAPPA, POT, ZA, ZB, ZC, 2>(W, K, rp, im, ip, jm, jp, km, kp, xcorr, gs, cs);
            else
                window_stencil<NDIRS, KAPPA, POT, ZA, ZB, ZC, 1>(W, K, rp, im, ip, jm, jp, km, kp, xcorr, gs, cs);
            if (FULL) {
                const float xv = XC[ZB];
                float d, htv, gv;
                if (CPA) {
                    asm volatile("cp.async.wait_group 3;" ::: "memory");   // voxel k's group (k+1..k+3 may pend)
                    const float* r = ring + ((k & 3) * 3) * nthr;
                    d = r[0];
                    gv = r[nthr];
                    htv = r[2 * nthr];
                } else {
                    d = Dv[Q];
                    gv = Gv[Q];
                    htv = Hv[Q];
                }
                const float s = fmaf(rho, htv, (1.f - rho) * gv);
                const float den = fmaf(rho, d, 2.f * cs);
                xnew = xv;
                if (den > 0.f) xnew = fminf(fmaxf(xv - fmaf(del, gs, s) * rcp_ftz(den), A.box_lo), A.box_hi);
                xn[idx] = xnew;
                if (!simple) A.ht[idx] = (1.f - alpha) * fmaf(d, xnew - xv, htv);
            } else {
                A.grad_out[idx] = del * gs;
                if (A.curv_out) A.curv_out[idx] = 2.f * cs;
            }
        }
        if (FULL && A.pfx) {
            CTR_CHECK(k >= 0 && k < G.nz, "update prefix staging");
            xs[k * 33 + lane] = xnew;
            run += xnew;
        }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    load_plane(I0(), k0 - 1);
    load_plane(I1(), k0);
    load_plane(I2(), k0 + 1);
    if (CPA) {
        issue_vox(k0);
        issue_vox(k0 + 1);
        issue_vox(k0 + 2);
    } else {
        load_vox(I1(), k0);
    }
    scale_plane(I0());
    scale_plane(I1());
    for (int k = k0; k < k1; k += 4) {
        step(I0(), I1(), I2(), I3(), k);
        if (k + 1 >= k1) break;
        step(I1(), I2(), I3(), I0(), k + 1);
        if (k + 2 >= k1) break;
        step(I2(), I3(), I0(), I1(), k + 2);
        if (k + 3 >= k1) break;
        step(I3(), I0(), I1(), I2(), k + 3);
    }
    if (UPD_DIAG & 2) return;   // timing diagnostic: no prefix write
    if (FULL && A.pfx) write_prefix(G, A.pfx, xs, tot, run, c, lane, act, col, k0, k1);
}

// Multi-GPU sub-iteration j: folds the all-reduced zeta of
// sub-iteration j-1 into g and htilde (Algorithm 1 lines 7-8 with rho_{j-2}),
// then runs lines 4-5 of sub-iteration j with rho_{j-1} from grad R(x) and D_R(x)
// computed by the UPD_STEN kernel while the all-reduce was in flight.  Elementwise
// (same block shape and z-prefix as k_update).  Ctl.k = j - 2 on entry (the
// advance follows this kernel); x buffers: in = A.xin, out = A.xa.
__global__ void __launch_bounds__(256) k_update_pre(DGeom G, const Ctl* __restrict__ ctl, UpdArgs A) {
    extern __shared__ float upd_sm[];
    const int lane = threadIdx.x, c = threadIdx.y, jj = threadIdx.z;
    const int NZC = blockDim.y;
    const int i = blockIdx.x * 32 + lane;
    const int j = blockIdx.y * blockDim.z + jj;
    const bool act = i < G.nx && j < G.ny;
    const float alpha = ctl->alpha;
    const float rho_f = rho_at(ctl, ctl->k), rho = rho_at(ctl, ctl->k + 1);
    const float inv_f = 1.f / (rho_f + 1.f);
    const unsigned col = act ? (unsigned)j * (unsigned)G.nx + (unsigned)i : 0u;
    const int k0 = c * A.CZ, k1 = min(G.nz, k0 + A.CZ);
    float* xs = upd_sm + (size_t)jj * G.nz * 33;
    float* tot = upd_sm + (size_t)blockDim.z * G.nz * 33 + (size_t)(jj * NZC) * 32;
    float run = 0.f;
    for (int k = k0; k < k1; k++) {
        float xnew = 0.f;
        if (act) {
            const unsigned idx = (unsigned)k * (unsigned)G.nxy + col;
            // lines 7-8 of sub-iteration j-1 (same arithmetic as the back-projection epilogue)
            const float z = __ldg(A.zeta + idx), gv = A.g[idx];
            const float gn = fmaf(rho_f * inv_f, fmaf(alpha, z, (1.f - alpha) * gv), gv * inv_f);
            const bool simple = ctl->simple;   // Algorithm 2: htilde holds zeta
            const float htv = simple ? z : fmaf(alpha, z, A.ht[idx]);
            A.g[idx] = gn;
            // lines 4-5 of sub-iteration j
            const float xv = __ldg(A.xin + idx), d = __ldg(A.dl + idx);
            const float s = fmaf(rho, htv, (1.f - rho) * gn);
            const float den = fmaf(rho, d, __ldg(A.curv + idx));
            xnew = xv;
            if (den > 0.f) xnew = fminf(fmaxf(xv - __fdividef(__ldg(A.grad + idx) + s, den), A.box_lo), A.box_hi);
            A.xa[idx] = xnew;
            A.ht[idx] = simple ? htv : (1.f - alpha) * fmaf(d, xnew - xv, htv);
        }
        if (A.pfx) {
            xs[k * 33 + lane] = xnew;
            run += xnew;
        }
    }
    if (A.pfx) write_prefix(G, A.pfx, xs, tot, run, c, lane, act, col, k0, k1);
}

// launch shape of the update kernels: NZC z-chunks of CZ voxels, JPB rows per block (<= 256 threads)
struct UpdShape {
    int nzc, cz, jpb;
    size_t smem;
};
static UpdShape upd_shape(const DGeom& G, bool pfx, bool ring = false) {
    UpdShape u;
    constexpr int zdiv = UPD_ZDIV;   // voxels per z-chunk target (tuning variants: -DUPD_ZDIV=n)
    u.nzc = std::min(8, std::max(1, G.nz / std::max(1, zdiv)));
    // at least 4 chunks once a column has 64 planes (c3: 4 x 16 instead of 2 x 32 planes, 0.086 ->
    // 0.077 ms, r2q; c4 keeps 4 x 24, c5 8 x 32)
    if (G.nz >= 64) u.nzc = std::max(u.nzc, 4);
    u.cz = (G.nz + u.nzc - 1) / u.nzc;
    u.nzc = (G.nz + u.cz - 1) / u.cz;
    u.jpb = std::max(1, 8 / u.nzc);  // JPB rows per block share x rows in L1
    u.smem = pfx ? sizeof(float) * ((size_t)u.jpb * G.nz * 33 + (size_t)u.jpb * u.nzc * 32) : 0;
    if (ring) u.smem += sizeof(float) * 4 * 3 * 256;   // UPD_CPA ring: [slot][D_L, g, htilde][256 threads]
    return u;
}

template <int POT, int NDIRS, bool KAPPA, int MODE>
static void upd_launch(const DGeom& G, const RegParams& rp, const Ctl* ctl, UpdArgs A, cudaStream_t s) {
    const UpdShape u = upd_shape(G, A.pfx != nullptr, MODE == UPD_FULL && UPD_CPA);
    A.CZ = u.cz;
    dim3 block(32, u.nzc, u.jpb), grid((G.nx + 31) / 32, (G.ny + u.jpb - 1) / u.jpb, 1);
    if (u.smem > 48 * 1024)
        cudaFuncSetAttribute(k_update<POT, NDIRS, KAPPA, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)u.smem);
    launch_k(k_update<POT, NDIRS, KAPPA, MODE>, grid, block, u.smem, s, G, rp, ctl, A);
}

template <int MODE>
static void upd_select(const DGeom& G, const RegParams& rp, const Ctl* ctl, const UpdArgs& A, cudaStream_t s) {
    const bool d4 = rp.n_dirs == 4, kp = A.kappa != nullptr;
#define CTR_UPD_CASE(POT)                                                              \
    if (d4) kp ? upd_launch<POT, 4, true, MODE>(G, rp, ctl, A, s) : upd_launch<POT, 4, false, MODE>(G, rp, ctl, A, s); \
    else kp ? upd_launch<POT, 13, true, MODE>(G, rp, ctl, A, s) : upd_launch<POT, 13, false, MODE>(G, rp, ctl, A, s);
    switch (rp.potential) {
        case 0: CTR_UPD_CASE(0) break;
        case 1: CTR_UPD_CASE(1) break;
        case 2: CTR_UPD_CASE(2) break;
        default: CTR_UPD_CASE(3) break;
    }
#undef CTR_UPD_CASE
}

void launch_reg(const DGeom& G, const RegParams& rp, const float* x, const float* kappa, float* grad, float* curv,
                cudaStream_t s, bool halo_lo, bool halo_hi) {
    UpdArgs A = {};
    A.xin = x;
    A.kappa = kappa;
    A.grad_out = grad;
    A.curv_out = curv;
    A.halo_lo = halo_lo;
    A.halo_hi = halo_hi;
    upd_select<UPD_STEN>(G, rp, nullptr, A, s);
    launches_add(1);
}

void launch_update(const DGeom& G, const RegParams& rp, const Ctl* ctl, float* xa, float* xb, const float* dl,
                   const float* g, float* ht, const float* kappa, float box_lo, float box_hi, float* pfx,
                   cudaStream_t s) {
    UpdArgs A = {};
    A.xa = xa;
    A.xb = xb;
    A.dl = dl;
    A.g = const_cast<float*>(g);
    A.ht = ht;
    A.kappa = kappa;
    A.pfx = pfx;
    A.box_lo = box_lo;
    A.box_hi = box_hi;
    upd_select<UPD_FULL>(G, rp, ctl, A, s);
    launches_add(1);
}

void launch_update_halo(const DGeom& G, const RegParams& rp, const Ctl* ctl, float* xa, float* xb, const float* dl,
                        float* g, float* ht, float box_lo, float box_hi, float* pfx, bool halo_lo, bool halo_hi,
                        cudaStream_t s, const float* kappa) {
    UpdArgs A = {};
    A.kappa = kappa;
    A.xa = xa;
    A.xb = xb;
    A.dl = dl;
    A.g = g;
    A.ht = ht;
    A.pfx = pfx;
    A.box_lo = box_lo;
    A.box_hi = box_hi;
    A.halo_lo = halo_lo;
    A.halo_hi = halo_hi;
    upd_select<UPD_FULL>(G, rp, ctl, A, s);
    launches_add(1);
}

void launch_update_pre(const DGeom& G, const Ctl* ctl, const float* xin, float* xout, const float* dl, float* g,
                       float* ht, const float* zeta, const float* grad, const float* curv, float box_lo,
                       float box_hi, float* pfx, cudaStream_t s) {
    UpdArgs A = {};
    A.xin = xin;
    A.xa = xout;
    A.dl = dl;
    A.g = g;
    A.ht = ht;
    A.zeta = zeta;
    A.grad = grad;
    A.curv = curv;
    A.pfx = pfx;
    A.box_lo = box_lo;
    A.box_hi = box_hi;
    const UpdShape u = upd_shape(G, pfx != nullptr);
    A.CZ = u.cz;
    dim3 block(32, u.nzc, u.jpb), grid((G.nx + 31) / 32, (G.ny + u.jpb - 1) / u.jpb, 1);
    if (u.smem > 48 * 1024)
        cudaFuncSetAttribute(k_update_pre, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)u.smem);
    k_update_pre<<<grid, block, u.smem, s>>>(G, ctl, A);
    launches_add(1);
}

// z-prefix of an arbitrary image (ct_forward_zprefix, the multi-GPU path after the all-gather):
// block = 32 columns of one row; its warps stage the planes in shared memory with coalesced loads
// (zs[k][column]) and write the columns with prefix_columns -- the same entries and rounding as
// write_prefix.  (UPD_PFXT = 0: thread = voxel column, P summed in k order.)
#if UPD_PFXT
__global__ void __launch_bounds__(256) k_zprefix(DGeom G, const float* __restrict__ x, float* __restrict__ pfx) {
    extern __shared__ float zp_sm[];   // zs[nz][33]
    const int lane = threadIdx.x, w = threadIdx.y, nw = blockDim.y;
    const int i0 = blockIdx.x * 32, j = blockIdx.y, i = i0 + lane;
    const float* __restrict__ xr = x + (size_t)j * G.nx + i;
    for (int k = w; k < G.nz; k += nw) zp_sm[k * 33 + lane] = i < G.nx ? __ldg(xr + (size_t)k * G.nxy) : 0.f;
    __syncthreads();
    prefix_columns(G, pfx, zp_sm, w, nw, lane, i0, j);
}

void launch_zprefix(const DGeom& G, const float* x, float* pfx, cudaStream_t s) {
    const size_t smem = sizeof(float) * 33 * (size_t)G.nz;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_zprefix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_zprefix<<<dim3((G.nx + 31) / 32, G.ny), dim3(32, 8), smem, s>>>(G, x, pfx);
    launches_add(1);
}
#else
__global__ void k_zprefix(DGeom G, const float* __restrict__ x, float* __restrict__ pfx) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= G.nxy) return;
    float2* __restrict__ pc = reinterpret_cast<float2*>(pfx) + (size_t)col * (size_t)pfx_stride_of(G);
    float P = 0.f;
    for (int k = 0; k < G.nz; k++) {
        const float xk = __ldg(x + (size_t)k * G.nxy + col);
        pc[k] = make_float2(fmaf(0.5f - (float)k, xk, P), xk);
        P += xk;
    }
    pc[G.nz] = make_float2(P, 0.f);
}

void launch_zprefix(const DGeom& G, const float* x, float* pfx, cudaStream_t s) {
    k_zprefix<<<(unsigned)((G.nxy + 127) / 128), 128, 0, s>>>(G, x, pfx);
    launches_add(1);
}
#endif

// ---- small elementwise kernels ----
__global__ void k_gh_update(long long n, const Ctl* __restrict__ ctl, const float* __restrict__ zeta, float* g,
                            float* ht) {
    const float rho = rho_of_k(ctl), alpha = ctl->alpha, inv = 1.f / (rho + 1.f);
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const float z = zeta[idx], gv = g[idx];
        g[idx] = fmaf(rho * inv, fmaf(alpha, z, (1.f - alpha) * gv), gv * inv);
        ht[idx] = ctl->simple ? z : fmaf(alpha, z, ht[idx]);
    }
}

__global__ void k_init_from_zeta(long long n, const float* __restrict__ zeta, float* g, float* ht) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        g[idx] = zeta[idx];
        ht[idx] = zeta[idx];
    }
}

__global__ void k_advance(Ctl* ctl, int n) {
    if ((int)threadIdx.x < n) ctl[threadIdx.x].k += 1;
}

// dst[i] = src[0][i] + src[1][i] + ... + src[n-1][i], src[p] = base + p * stride, summed in rank
// order (deterministic): the single-process emulation of the partial-gradient reduction
__global__ void k_sum_partials(float* __restrict__ base, int n, long long stride, long long count) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        float acc = base[i];
        for (int p = 1; p < n; p++) acc += __ldg(base + p * stride + i);
        base[i] = acc;
    }
}

__global__ void k_fill(float* p, long long n, float v) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x)
        p[idx] = v;
}

// kappa_j = sqrt([A'W1]_j / [A'1]_j), 0/0 = 1
__global__ void k_kappa_ratio(long long n, const float* __restrict__ a, const float* __restrict__ b, float* kappa) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const float bv = b[idx];
        kappa[idx] = bv > 0.f ? sqrtf(a[idx] / bv) : 1.f;
    }
}

__global__ void k_state_h(long long n, const float* __restrict__ dl, const float* __restrict__ x,
                          const float* __restrict__ ht, float* h) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x)
        h[idx] = fmaf(dl[idx], x[idx], -ht[idx]);
}

__global__ void k_check(long long n, const float* __restrict__ x, const float* __restrict__ xref, int* flag,
                        double* dsum) {
    double acc = 0.0;
    int bad = 0;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const float v = x[idx];
        if (!isfinite(v)) bad = 1;
        if (xref) {
            const double d = (double)v - (double)xref[idx];
            acc += d * d;
        }
    }
    // warp reduce then one atomic per warp (a scalar diagnostic, not the data path)
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_down_sync(0xffffffffu, acc, o);
        bad |= __shfl_down_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicOr(flag, 1);
        if (xref) atomicAdd(dsum, acc);
    }
}

static int grid_for(long long n) {
    long long b = (n + 255) / 256;
    return (int)(b < 148LL * 16 ? b : 148LL * 16);
}

void launch_gh_update(const DGeom& G, const Ctl* ctl, const float* zeta, float* g, float* ht, cudaStream_t s) {
    k_gh_update<<<grid_for(G.nvox), 256, 0, s>>>(G.nvox, ctl, zeta, g, ht);
    launches_add(1);
}
void launch_init_from_zeta(const DGeom& G, const float* zeta, float* g, float* ht, cudaStream_t s) {
    k_init_from_zeta<<<grid_for(G.nvox), 256, 0, s>>>(G.nvox, zeta, g, ht);
    launches_add(1);
}
void launch_fill(float* p, long long n, float v, cudaStream_t s) {
    k_fill<<<grid_for(n), 256, 0, s>>>(p, n, v);
    launches_add(1);
}
void launch_kappa_ratio(long long n, const float* a, const float* b, float* kappa, cudaStream_t s) {
    k_kappa_ratio<<<grid_for(n), 256, 0, s>>>(n, a, b, kappa);
    launches_add(1);
}
void launch_advance(Ctl* ctl, cudaStream_t s, int n) {
    k_advance<<<1, 32, 0, s>>>(ctl, n);
    launches_add(1);
}
void launch_sum_partials(float* base, int n, long long stride, long long count, cudaStream_t s) {
    k_sum_partials<<<grid_for(count), 256, 0, s>>>(base, n, stride, count);
    launches_add(1);
}
void launch_state_h(const DGeom& G, const float* dl, const float* x, const float* ht, float* h, cudaStream_t s) {
    k_state_h<<<grid_for(G.nvox), 256, 0, s>>>(G.nvox, dl, x, ht, h);
    launches_add(1);
}
void launch_check(const DGeom& G, const float* x, const float* xref, int* flag, double* dsum, cudaStream_t s) {
    k_check<<<grid_for(G.nvox), 256, 0, s>>>(G.nvox, x, xref, flag, dsum);
    launches_add(1);
}

}  // namespace ctr
