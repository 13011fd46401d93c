// proj_fwd.cu — K1+K2: ray-driven separable-footprint forward projection with
// the statistically weighted residual fused in the epilogue.
//
// Gathers over the fan wedge of a group of detector columns (2-D: k_fwd2,
// 3-D: k_fwd3, described at each kernel); both test candidate voxel columns
// against the wedge's edge rays and evaluate the SF footprint with
// ct_footprint, the function the back-projector uses.  No atomics.
//
// Epilogue (Eq. 36 applied implicitly):
//   FWD_PLAIN  p = L_z q
//   FWD_RESID  r = L_z w (L_z q - y)     -> back-projector needs no L_z
//   FWD_ONES_W r = L_z w (L_z A0 1)      (D_L = A'WA1)
#include <algorithm>
#include <cmath>
#include <vector>

#include "kernels.cuh"

namespace ctr {

// ---------------------------------------------------------------------------
// 2-D forward projection.  A warp owns F2_CPW = 8 adjacent detector cells
// s0..s0+7 of one view and walks the union of their fan wedges along the
// dominant axis, F2_SPP = 4 slabs per pass: the 8 lanes of a slab split its
// candidate pixels (support-function test of the pixel square against the two
// union edge rays), evaluate the SF footprint (ct_footprint, shared with the
// back-projector), F1 of the 8 cells from 9 edge evaluations of the trapezoid
// antiderivative, and accumulate L_xy F1 x into 8 per-lane registers.  A warp
// reduction forms the 8 sums; no atomics, no shared memory.
#ifndef F2_SPLIT_W
#define F2_SPLIT_W 4   // warps sharing one 8-cell group (each walks every F2_SPLIT-th slab batch)
#endif
constexpr int F2_CPW = 8;
constexpr int F2_SUB = 8;            // lanes per slab
constexpr int F2_SPP = 32 / F2_SUB;  // slabs per pass
constexpr int F2_WARPS = 4;
constexpr int F2_SPLIT = F2_SPLIT_W;
constexpr int F2_GPB = F2_WARPS / F2_SPLIT;   // cell groups per block

template <bool ARC, int MODE>
__global__ void __launch_bounds__(32 * F2_WARPS)
k_fwd2(DGeom G, const float4* __restrict__ vtab, const Ctl* __restrict__ ctl, Views vsel,
       const float* __restrict__ xa, const float* __restrict__ xb, const float* __restrict__ y,
       const float* __restrict__ w, float* __restrict__ out) {
    pdl_enter();
    constexpr bool ONES = (MODE == FWD_ONES_W);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const Views V = select_views(ctl, vsel);
    const int vi = blockIdx.y;
    if (vi >= V.count) return;
    const int v = V.start + vi * V.stride;
    const int grp = wid / F2_SPLIT, part = wid % F2_SPLIT;   // cell group, slab-batch residue
    const int s0 = (blockIdx.x * F2_GPB + grp) * F2_CPW;
    __shared__ float red[F2_WARPS][F2_CPW];
    const float* __restrict__ x = xa;
    if (ctl) x = (((ctl->k - ctl->k_base) & 1) != 0) ? xa : xb;
    const float4 vw = __ldg(&vtab[v]);
    const float cb = vw.x, sb = vw.y;
    const float Sx = G.dso * cb, Sy = G.dso * sb;
    float acc[F2_CPW];
#pragma unroll
    for (int c = 0; c < F2_CPW; c++) acc[c] = 0.f;

    const int s7 = min(s0 + F2_CPW - 1, G.ns - 1);
    const float tl = ((float)s0 - 0.5f - G.s_c0) * G.delta;
    const float tr = ((float)s7 + 0.5f - G.s_c0) * G.delta;
    const float tm = (0.5f * (float)(s0 + s7) - G.s_c0) * G.delta;
    float cal, cul, car, cur_, cam, cum;
    if (ARC) {
        sincosf(tl, &cul, &cal);
        sincosf(tr, &cur_, &car);
        sincosf(tm, &cum, &cam);
    } else {
        cal = car = cam = G.dsd;
        cul = tl; cur_ = tr; cum = tm;
    }
    // world directions d = ca e_c + cu e_u, e_c = (-cb, -sb), e_u = (-sb, cb)
    const float dlx = -cal * cb - cul * sb, dly = -cal * sb + cul * cb;
    const float drx = -car * cb - cur_ * sb, dry = -car * sb + cur_ * cb;
    const float dmx = -cam * cb - cum * sb, dmy = -cam * sb + cum * cb;
    // inward normals: tau > tau_l <=> nl.(P-S) > 0 ; tau < tau_r <=> nr.(P-S) > 0
    const float nlx = -cal * sb + cul * cb, nly = cal * cb + cul * sb;
    const float nrx = car * sb - cur_ * cb, nry = -car * cb - cur_ * sb;
    const float hx = 0.5f * G.dx, hy = 0.5f * G.dy;
    const float suppl = fabsf(nlx) * hx + fabsf(nly) * hy;
    const float suppr = fabsf(nrx) * hx + fabsf(nry) * hy;
    const float tol_l = 1e-4f * suppl, tol_r = 1e-4f * suppr;
    const bool xstep = fabsf(dmx) >= fabsf(dmy);
    const int na_ = xstep ? G.nx : G.ny, no_ = xstep ? G.ny : G.nx;
    const float a0 = xstep ? G.x0 : G.y0, da = xstep ? G.dx : G.dy, ha = xstep ? hx : hy;
    const float o0 = xstep ? G.y0 : G.x0, dob = xstep ? G.dy : G.dx;
    const float Sa = xstep ? Sx : Sy, So = xstep ? Sy : Sx;
    const float kl = xstep ? dly / dlx : dlx / dly;
    const float kr = xstep ? dry / drx : drx / dry;
    const float sgn = (xstep ? dlx : dly) > 0.f ? 1.f : -1.f;
    const float inv_do = 1.f / dob;

    for (int sl0 = part * F2_SPP; s0 < G.ns && sl0 < na_; sl0 += F2_SPP * F2_SPLIT) {
        const int sl = sl0 + lane / F2_SUB, sub = lane % F2_SUB;
        int lo = 0, hi = -1;
        if (sl < na_) {
            const float ac = fmaf((float)sl, da, a0);
            const float pa = ac - ha - Sa, pb = ac + ha - Sa;
            if (pa * sgn > 0.f && pb * sgn > 0.f) {
                const float y1 = fmaf(pa, kl, So), y2 = fmaf(pb, kl, So);
                const float y3 = fmaf(pa, kr, So), y4 = fmaf(pb, kr, So);
                const float f0 = (fminf(fminf(y1, y2), fminf(y3, y4)) - o0) * inv_do + 0.5f;
                const float f1 = (fmaxf(fmaxf(y1, y2), fmaxf(y3, y4)) - o0) * inv_do + 0.5f;
                if (f1 >= -1.f && f0 <= (float)no_ + 1.f) {
                    lo = max((int)floorf(f0 - 1e-3f), 0);
                    hi = min((int)floorf(f1 + 1e-3f), no_ - 1);
                }
            }
        }
        const int npass = __reduce_max_sync(0xffffffffu, (hi - lo + F2_SUB) / F2_SUB);
        for (int p = 0; p < npass; p++) {
            const int o = lo + sub + F2_SUB * p;
            if (o > hi) continue;
            const int i = xstep ? sl : o, j = xstep ? o : sl;
            const float cx = fmaf((float)i, G.dx, G.x0) - Sx;
            const float cy = fmaf((float)j, G.dy, G.y0) - Sy;
            if (fmaf(nlx, cx, nly * cy) + suppl < -tol_l || fmaf(nrx, cx, nry * cy) + suppr < -tol_r) continue;
            Footprint f;
            ct_footprint<ARC>(G, cb, sb, 0.f, i, j, f);
            const float Lx = f.lxy * (ONES ? 1.f : __ldg(&x[(size_t)j * G.nx + i]));
            float T0 = trap_T(f, ((float)s0 - 0.5f) - f.sfc);
#pragma unroll
            for (int c = 0; c < F2_CPW; c++) {
                const float T1 = trap_T(f, ((float)(s0 + c) + 0.5f) - f.sfc);
                acc[c] = fmaf(Lx, T1 - T0, acc[c]);
                T0 = T1;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < F2_CPW; c++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    }
    // sum the F2_SPLIT warps of the cell group (fixed order: deterministic)
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < F2_CPW; c++) red[wid][c] = acc[c];
    }
    __syncthreads();
    if (part != 0 || s0 >= G.ns) return;
    float q = 0.f;
    if (lane < F2_CPW) {
        for (int pw = 0; pw < F2_SPLIT; pw++) q += red[grp * F2_SPLIT + pw][lane];
    }
    const int s = s0 + lane;
    if (lane < F2_CPW && s < G.ns) {
        const size_t o = (size_t)vi * G.ns + s;
        if (MODE == FWD_PLAIN) {
            out[o] = q;
        } else {
            const size_t a = (size_t)v * G.ns + s;
            const float wv = w ? __ldg(&w[a]) : 1.f;
            if (MODE == FWD_RESID) out[o] = wv * (q - __ldg(&y[a]));
            else out[o] = wv * q;
        }
    }
}

// ---------------------------------------------------------------------------
// 2-D forward projection, block-wide cell groups (k_fwd2b, the default; F2B = 0 selects k_fwd2
// above).  A block of F2B_WARPS warps owns CPB = 16 or 32 adjacent detector cells of one view and
// walks the union of their fan wedges; the warps take interleaved slab passes (F2B_SUB lanes per
// slab split its candidate pixels).  Each candidate pixel's footprint is evaluated once for the
// whole block (k_fwd2 evaluated it once per 8-cell warp group, ~1.25 times per pixel-view at c2)
// and F1 only for the cells under it (nc + 1 antiderivative evaluations instead of 9); the credits
// L_xy F1 x go to the lane's own row of a shared-memory tile [warp][lane][CPB + 1] (no atomics),
// which is summed over lanes and warps in a fixed order at the end (deterministic).
#ifndef F2B
#define F2B 1
#endif
#ifndef F2B_CPB
#define F2B_CPB 0      // cells per block: 0 = chosen per launch (32 / 16 / 8), else forced
#endif
#ifndef F2B_MINBPS
#define F2B_MINBPS 4   // the widest group that still gives this many blocks per SM
#endif
#ifndef F2B_LPS
#define F2B_LPS 2      // lanes per slab (measured c2: 2 > 4 > 8 > 16, profiles/r2s/fwd2b_ab.log)
#endif
constexpr int F2B_SUB = F2B_LPS;           // lanes per slab
constexpr int F2B_SPP = 32 / F2B_SUB;      // slabs per warp pass

// F2B_WARPS warps per block: 8 for 32-cell groups (c2), 4 for 16 / 8 (c1) -- measured
template <bool ARC, int MODE, int CPB, int F2B_WARPS>
__global__ void __launch_bounds__(32 * F2B_WARPS)
k_fwd2b(DGeom G, const float4* __restrict__ vtab, const Ctl* __restrict__ ctl, Views vsel,
        const float* __restrict__ xa, const float* __restrict__ xb, const float* __restrict__ y,
        const float* __restrict__ w, float* __restrict__ out) {
    pdl_enter();
    constexpr bool ONES = (MODE == FWD_ONES_W);
    __shared__ float rows[F2B_WARPS * 32 * (CPB + 1)];
    __shared__ float wsum[F2B_WARPS][CPB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float* __restrict__ row = rows + (wid * 32 + lane) * (CPB + 1);
#pragma unroll
    for (int c = 0; c < CPB; c++) row[c] = 0.f;
    const Views V = select_views(ctl, vsel);
    const int vi = blockIdx.y;
    if (vi >= V.count) return;   // block-uniform
    const int v = V.start + vi * V.stride;
    const int s0 = blockIdx.x * CPB;
    const float* __restrict__ x = xa;
    if (ctl) x = (((ctl->k - ctl->k_base) & 1) != 0) ? xa : xb;
    const float4 vw = __ldg(&vtab[v]);
    const float cb = vw.x, sb = vw.y;
    const float Sx = G.dso * cb, Sy = G.dso * sb;
    const int slast = min(s0 + CPB - 1, G.ns - 1);
    const float tl = ((float)s0 - 0.5f - G.s_c0) * G.delta;
    const float tr = ((float)slast + 0.5f - G.s_c0) * G.delta;
    const float tm = (0.5f * (float)(s0 + slast) - G.s_c0) * G.delta;
    float cal, cul, car, cur_, cam, cum;
    if (ARC) {
        sincosf(tl, &cul, &cal);
        sincosf(tr, &cur_, &car);
        sincosf(tm, &cum, &cam);
    } else {
        cal = car = cam = G.dsd;
        cul = tl; cur_ = tr; cum = tm;
    }
    const float dlx = -cal * cb - cul * sb, dly = -cal * sb + cul * cb;
    const float drx = -car * cb - cur_ * sb, dry = -car * sb + cur_ * cb;
    const float dmx = -cam * cb - cum * sb, dmy = -cam * sb + cum * cb;
    const float nlx = -cal * sb + cul * cb, nly = cal * cb + cul * sb;
    const float nrx = car * sb - cur_ * cb, nry = -car * cb - cur_ * sb;
    const float hx = 0.5f * G.dx, hy = 0.5f * G.dy;
    const float suppl = fabsf(nlx) * hx + fabsf(nly) * hy;
    const float suppr = fabsf(nrx) * hx + fabsf(nry) * hy;
    const float tol_l = 1e-4f * suppl, tol_r = 1e-4f * suppr;
    const bool xstep = fabsf(dmx) >= fabsf(dmy);
    const int na_ = xstep ? G.nx : G.ny, no_ = xstep ? G.ny : G.nx;
    const float a0 = xstep ? G.x0 : G.y0, da = xstep ? G.dx : G.dy, ha = xstep ? hx : hy;
    const float o0 = xstep ? G.y0 : G.x0, dob = xstep ? G.dy : G.dx;
    const float Sa = xstep ? Sx : Sy, So = xstep ? Sy : Sx;
    const float kl = xstep ? dly / dlx : dlx / dly;
    const float kr = xstep ? dry / drx : drx / dry;
    const float sgn = (xstep ? dlx : dly) > 0.f ? 1.f : -1.f;
    const float inv_do = 1.f / dob;
    __syncwarp();

    for (int sl0 = wid * F2B_SPP; sl0 < na_; sl0 += F2B_SPP * F2B_WARPS) {
        const int sl = sl0 + lane / F2B_SUB, sub = lane % F2B_SUB;
        int lo = 0, hi = -1;
        if (sl < na_) {
            const float ac = fmaf((float)sl, da, a0);
            const float pa = ac - ha - Sa, pb = ac + ha - Sa;
            if (pa * sgn > 0.f && pb * sgn > 0.f) {
                const float y1 = fmaf(pa, kl, So), y2 = fmaf(pb, kl, So);
                const float y3 = fmaf(pa, kr, So), y4 = fmaf(pb, kr, So);
                const float f0 = (fminf(fminf(y1, y2), fminf(y3, y4)) - o0) * inv_do + 0.5f;
                const float f1 = (fmaxf(fmaxf(y1, y2), fmaxf(y3, y4)) - o0) * inv_do + 0.5f;
                if (f1 >= -1.f && f0 <= (float)no_ + 1.f) {
                    lo = max((int)floorf(f0 - 1e-3f), 0);
                    hi = min((int)floorf(f1 + 1e-3f), no_ - 1);
                }
            }
        }
        const int npass = __reduce_max_sync(0xffffffffu, (hi - lo + F2B_SUB) / F2B_SUB);
        for (int p = 0; p < npass; p++) {
            const int o = lo + sub + F2B_SUB * p;
            if (o > hi) continue;
            const int i = xstep ? sl : o, j = xstep ? o : sl;
            const float cx = fmaf((float)i, G.dx, G.x0) - Sx;
            const float cy = fmaf((float)j, G.dy, G.y0) - Sy;
            if (fmaf(nlx, cx, nly * cy) + suppl < -tol_l || fmaf(nrx, cx, nry * cy) + suppr < -tol_r) continue;
            Footprint f;
            ct_footprint<ARC>(G, cb, sb, 0.f, i, j, f);
            // cells under the footprint within the block's cells (the back-projector's range)
            const int slo = max((int)floorf(f.sfc + f.u0 + 0.5f), s0);
            const int shi = min((int)floorf(f.sfc + f.u3 + 0.5f), slast);
            if (slo > shi) continue;
            const float Lx = f.lxy * (ONES ? 1.f : __ldg(&x[(size_t)j * G.nx + i]));
            float T0 = trap_T(f, ((float)slo - 0.5f) - f.sfc);
            for (int sc = slo; sc <= shi; sc++) {
                const float T1 = trap_T(f, ((float)sc + 0.5f) - f.sfc);
                CTR_CHECK(sc - s0 >= 0 && sc - s0 < CPB, "fwd2b cell");
                row[sc - s0] = fmaf(Lx, T1 - T0, row[sc - s0]);
                T0 = T1;
            }
        }
    }
    // cell c: the 32 lane rows of each warp in lane order, then the warps in order
    __syncwarp();
    for (int c = lane; c < CPB; c += 32) {
        float q = 0.f;
        const float* __restrict__ col = rows + wid * 32 * (CPB + 1) + c;
#pragma unroll 8
        for (int l = 0; l < 32; l++) q += col[l * (CPB + 1)];
        wsum[wid][c] = q;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < CPB; c += 32 * F2B_WARPS) {
        const int sc = s0 + c;
        float q = 0.f;
#pragma unroll
        for (int pw = 0; pw < F2B_WARPS; pw++) q += wsum[pw][c];
        if (sc < G.ns) {
            const size_t o = (size_t)vi * G.ns + sc;
            if (MODE == FWD_PLAIN) {
                out[o] = q;
            } else {
                const size_t a = (size_t)v * G.ns + sc;
                const float wv = w ? __ldg(&w[a]) : 1.f;
                if (MODE == FWD_RESID) out[o] = wv * (q - __ldg(&y[a]));
                else out[o] = wv * q;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 3-D forward projection.  A warp owns F3_CPW = 4 adjacent detector columns
// s0..s0+3 of one view (the union of their fan wedges); lane l owns the RPL
// consecutive detector rows t = RPL*l + r of all four columns.  The warp walks
// the union wedge 8 slabs at a time: lanes split the candidate voxel columns
// (4 per slab per pass), test the column's magnified axial extent against the
// detector rows first (helical views near the ends of the helix reach few
// rows), evaluate the transaxial footprints in parallel (ct_internal.cuh,
// shared with the back-projector; F1 for the four detector columns) and push
// the voxel columns with any F1 > 0 into a warp queue (ballot + prefix
// popcount).  Each queued voxel column is resampled onto the rows once and
// credited to the four detector columns with their own L = L_xy F1 (a voxel
// column's footprint covers ~2.4 detector columns, so this removes most of the
// redundant resampling of a one-column-per-warp walk).
//   PFX (solve path): the x-update writes (A_k, x_k), A_k = P_k - (k - 1/2) x_k
//     with P_k = sum_{k'<k} x_k', of every voxel column (float2, z-fastest,
//     stride pfx_stride).  The magnified column is a piecewise-linear cumulative
//     X(u) = H (P_k + (f' - k + 1/2) x_k) = H (A_k + f' x_k) over row units u
//     (f' the voxel coordinate, k = round(f')), and
//     the exact F2-weighted row sum is X(t+1) - X(t): RPL interpolations (one
//     8-byte gather each) per lane plus one shuffle, no per-voxel loop, no
//     divergence.
//   direct (ct_forward / init / D_L): row t loops over the voxels whose
//     magnified extent [b_k, b_k+1] meets [t, t+1] (same overlap arithmetic as
//     the back-projector), reading x in the boundary layout.
// No atomics; row sums live in registers; the epilogue stages the block's 32
// detector columns through shared memory so y/w reads and r writes are
// 128-byte runs.
#ifndef F3_NWARPS
#define F3_NWARPS 4    // warps per block (4 detector columns each)
#endif
#ifndef F3_SUB
#define F3_SUB 1       // lanes per slab in the candidate walk (32 / F3_SUB slabs per pass)
#endif
constexpr int F3_WARPS = F3_NWARPS;
constexpr int F3_CPW = 4;
constexpr int F3_CPB = F3_WARPS * F3_CPW;   // detector columns per block

// Experiment: F3_TMA = 1 stages each queued hit's run of z-prefix entries in shared
// memory with a 1-D bulk copy (cp.async.bulk, the TMA engine) F3_TMAD hits ahead, completion
// signalled on a per-slot mbarrier; the hit loop then reads the run from shared memory instead
// of gathering from L2 / HBM.
#ifndef F3_TMA
#define F3_TMA 0
#endif
#ifndef F3_TMAD
#define F3_TMAD 3      // bulk-copy ring depth (hits in flight per warp)
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok)
                     : "r"(bar), "r"(parity)
                     : "memory");
    } while (!ok);
}
// one lane: copy `bytes` (multiple of 16, both addresses 16-byte aligned) from global to shared,
// completion counted on the barrier
__device__ __forceinline__ void bulk_copy(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

#ifndef F3_VIEWCULL
#define F3_VIEWCULL 1  // skip the walk of views whose cone misses the volume (thin z-slabs)
#endif
#ifndef F3_CREDIT2
#define F3_CREDIT2 0   // a hit's credits to the 4 detector columns as packed FP32 pairs (FFMA2)
#endif
#ifndef F3_WCSMEM
#define F3_WCSMEM 1    // the candidate walk's per-warp constants in shared memory (frees registers)
#endif
struct WalkC {
    float nlx, nly, nrx, nry, suppl, suppr, tol_l, tol_r, kl, kr, Sa, So, a0, da, ha, o0, inv_do, sgn, Sx, Sy, cb, sb,
        zs;
    int na_, no_;
    bool xstep;
};
#ifndef F3_SUNROLL
#define F3_SUNROLL 8   // hit-loop unroll (8: c4 fwd 2.51 -> 2.31 ms with F3_WCSMEM, r2o)
#endif
#ifndef F3_STRIDED
#define F3_STRIDED 0   // lane l owns detector rows RPL l + r (0) or l + 32 r (1)
#endif
constexpr int kF3SingleUnroll = F3_SUNROLL;
// Detector row r of lane l.  The strided assignment (l + 32 r: each gather instruction covers 32
// consecutive rows, about half the cache lines of the consecutive one) measured slower (c4 fwd
// 2.60 vs 2.51 ms, r2h) and is kept as a tuning switch only.
template <int RPL>
__device__ __forceinline__ int fwd_row(int lane, int r) { return F3_STRIDED ? lane + 32 * r : RPL * lane + r; }
#ifndef F3_PREYW
#define F3_PREYW 1     // epilogue y, w copied into shared memory by cp.async at kernel start
#endif
#ifndef F3_MINB
#define F3_MINB 8  // 64 registers: 8 blocks of 4 warps per SM to hide the prefix-gather latency
#endif
// NW warps per block (4, or 2 for small grids: finer blocks shorten the last wave); 32 / NW
// blocks per SM keep the same 32 resident warps at 64 registers
// SEG (segmented forward, c5-sized volumes whose z-prefix exceeds L2): block b
// takes its (view, detector-column block, segment) from sched[b] -- entries sorted by the xy tile
// the segment's piece of the wedge crosses, so that resident blocks share a tile's z-prefix in
// L2 -- walks only the segment's slabs [seg * seg_len, (seg + 1) * seg_len) and writes its raw row
// sums to part[seg][vi][t][s]; k_fwd3_reduce adds the segments in order and applies the epilogue.
template <bool ARC, int MODE, int RPL, bool PFX, int NW, bool SEG = false>
__global__ void __launch_bounds__(32 * NW, F3_MINB * F3_NWARPS / NW)
k_fwd3(DGeom G, const float4* __restrict__ vtab, const Ctl* __restrict__ ctl, Views vsel,
       const float* __restrict__ xa, const float* __restrict__ xb, const float* __restrict__ y,
       const float* __restrict__ w, float* __restrict__ out, int pfx_stride, int slot_entries,
       const int2* __restrict__ sched, int seg_len, int part_views) {
    pdl_enter();
    constexpr bool TMA = PFX && F3_TMA;
    constexpr int TD = F3_TMAD;
    extern __shared__ __align__(16) float2 fwd_ring[];   // TMA: [NW][TD][slot_entries]
    __shared__ __align__(8) unsigned long long fbar[TMA ? NW : 1][TMA ? TD : 1];
    __shared__ int2 qR[TMA ? NW : 1][32];   // TMA: (global element offset of the run, first entry | entries << 16)
#if F3_WCSMEM
    __shared__ WalkC wcs[NW];
#endif
    __shared__ float4 qL[NW][32];    // L for the 4 detector columns
    __shared__ float4 qG[NW][32];    // PFX: (1/(H nz), -B0/(H nz), column offset, X(top)); direct: (B0, H, col, -)
    __shared__ float stage[32 * RPL][(NW * F3_CPW) + 1];
#if F3_PREYW
    __shared__ float ysm[MODE == FWD_RESID ? 32 * RPL : 1][(NW * F3_CPW)];   // epilogue operands (cp.async)
    __shared__ float wsm[MODE != FWD_PLAIN ? 32 * RPL : 1][(NW * F3_CPW)];
#endif
    constexpr bool ONES = (MODE == FWD_ONES_W);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const Views V = select_views(ctl, vsel);
    int vi = blockIdx.y, bxi = blockIdx.x, seg = 0;
    if (SEG) {
        const int2 e = __ldg(&sched[blockIdx.x]);
        vi = e.x;
        bxi = e.y & 0xffff;
        seg = e.y >> 16;
    }
    if (vi >= V.count) return;
    const int v = V.start + vi * V.stride;
    const int sb0 = bxi * (NW * F3_CPW);          // first detector column of the block
    const int s0 = sb0 + wid * F3_CPW;             // first detector column of the warp
    const float* __restrict__ x = xa;
    if (ctl && !PFX) x = (((ctl->k - ctl->k_base) & 1) != 0) ? xa : xb;
    const float2* __restrict__ Q = reinterpret_cast<const float2*>(xa);  // PFX: z-prefix array
    const float4 vw = __ldg(&vtab[v]);
    const float cb = vw.x, sb = vw.y, zs = vw.z;
    const float Sx = G.dso * cb, Sy = G.dso * sb;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    unsigned tcnt = 0;   // TMA: bulk copies consumed by this warp (ring slot and phase)
    if (TMA) {
        if (lane == 0) {
            for (int q = 0; q < TD; q++) mbar_init(smem_u32(&fbar[wid][q]));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }

#if F3_CREDIT2
    // row sums of detector columns (0, 1) and (2, 3) as packed pairs: a hit's credits are 2 RPL
    // FFMA2 (L4.xy / L4.zw times the broadcast row sum) instead of 4 RPL FFMA
    float2 acc2[2][RPL];
#pragma unroll
    for (int c = 0; c < 2; c++)
#pragma unroll
        for (int r = 0; r < RPL; r++) acc2[c][r] = make_float2(0.f, 0.f);
#else
    float acc[F3_CPW][RPL];
#pragma unroll
    for (int c = 0; c < F3_CPW; c++)
#pragma unroll
        for (int r = 0; r < RPL; r++) acc[c][r] = 0.f;
#endif

#if F3_PREYW
    // y and w of the block's (row, column) outputs are read only by the epilogue: start their
    // copies into shared memory now (cp.async) so that the epilogue does not wait on HBM
    constexpr bool YW = (MODE != FWD_PLAIN) && !SEG;
    if (YW) {
        for (int q = threadIdx.x; q < G.nt * (NW * F3_CPW); q += (32 * NW)) {
            const int t = q / (NW * F3_CPW), c = q % (NW * F3_CPW);
            const int ss = sb0 + c;
            if (ss >= G.ns) continue;
            const size_t a = ((size_t)v * G.nt + t) * G.ns + ss;
            if (MODE == FWD_RESID)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                 (unsigned)__cvta_generic_to_shared(&ysm[t][c])),
                             "l"(__cvta_generic_to_global(y + a))
                             : "memory");
            if (w)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                 (unsigned)__cvta_generic_to_shared(&wsm[t][c])),
                             "l"(__cvta_generic_to_global(w + a))
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
#endif

    // view cull (block-uniform): the voxel columns span detector rows [(zbot - z_s) m + t_c0p,
    // (ztop - z_s) m + t_c0p] for a magnification m (rows per mm) in [mlo, mhi]; a view whose cone
    // misses the volume (helical views beyond a thin z-slab, the ends of a long helix) projects to 0
    // and skips the walk (the epilogue still writes its outputs)
    bool reach = true;
    if (F3_VIEWCULL) {
        const float mlo = G.dsd / (G.dso + G.rxy) * G.inv_dt, mhi = G.dsd / (G.dso - G.rxy) * G.inv_dt;
        const float za = G.zbot - zs, zb = G.ztop - zs;
        reach = fminf(za * mlo, za * mhi) + G.t_c0p < (float)G.nt + 1.f && fmaxf(zb * mlo, zb * mhi) + G.t_c0p > -1.f;
    }
    if (s0 < G.ns && reach) {  // warp-uniform
        const int s3 = min(s0 + F3_CPW - 1, G.ns - 1);
        const float tl = ((float)s0 - 0.5f - G.s_c0) * G.delta;
        const float tr = ((float)s3 + 0.5f - G.s_c0) * G.delta;
        const float tm = (0.5f * (float)(s0 + s3) - G.s_c0) * G.delta;
        float cal, cul, car, cur_, cam, cum;
        if (ARC) {
            sincosf(tl, &cul, &cal);
            sincosf(tr, &cur_, &car);
            sincosf(tm, &cum, &cam);
        } else {
            cal = car = cam = G.dsd;
            cul = tl; cur_ = tr; cum = tm;
        }
        const float dlx = -cal * cb - cul * sb, dly = -cal * sb + cul * cb;
        const float drx = -car * cb - cur_ * sb, dry = -car * sb + cur_ * cb;
        const float dmx = -cam * cb - cum * sb, dmy = -cam * sb + cum * cb;
        const float nlx = -cal * sb + cul * cb, nly = cal * cb + cul * sb;
        const float nrx = car * sb - cur_ * cb, nry = -car * cb - cur_ * sb;
        const float hx = 0.5f * G.dx, hy = 0.5f * G.dy;
        const float suppl = fabsf(nlx) * hx + fabsf(nly) * hy;
        const float suppr = fabsf(nrx) * hx + fabsf(nry) * hy;
        const float tol_l = 1e-4f * suppl, tol_r = 1e-4f * suppr;
        const bool xstep = fabsf(dmx) >= fabsf(dmy);
        // stepping axis "a" (slabs) and other axis "o"
        const int na_ = xstep ? G.nx : G.ny, no_ = xstep ? G.ny : G.nx;
        const float a0 = xstep ? G.x0 : G.y0, da = xstep ? G.dx : G.dy, ha = xstep ? hx : hy;
        const float o0 = xstep ? G.y0 : G.x0, dob = xstep ? G.dy : G.dx;
        const float Sa = xstep ? Sx : Sy, So = xstep ? Sy : Sx;
        const float kl = xstep ? dly / dlx : dlx / dly;
        const float kr = xstep ? dry / drx : drx / dry;
        const float sgn = (xstep ? dlx : dly) > 0.f ? 1.f : -1.f;
        const float inv_do = 1.f / dob;
        const float fnz = (float)G.nz, rnz = 1.f / (float)G.nz;
#if F3_WCSMEM
        // the walk's per-warp constants live in shared memory (volatile reads in the producer) so that
        // they do not hold registers through the hit loop
        if (lane == 0) {
            volatile WalkC* wv = &wcs[wid];
            wv->nlx = nlx; wv->nly = nly; wv->nrx = nrx; wv->nry = nry; wv->suppl = suppl; wv->suppr = suppr;
            wv->tol_l = tol_l; wv->tol_r = tol_r; wv->kl = kl; wv->kr = kr; wv->Sa = Sa; wv->So = So;
            wv->a0 = a0; wv->da = da; wv->ha = ha; wv->o0 = o0; wv->inv_do = inv_do; wv->sgn = sgn;
            wv->Sx = Sx; wv->Sy = Sy; wv->na_ = na_; wv->no_ = no_; wv->xstep = xstep; wv->cb = cb; wv->sb = sb;
            wv->zs = zs;
        }
        __syncwarp();
        const volatile WalkC* wcv = &wcs[wid];
#define WCX(v) (wcv->v)
#else
#define WCX(v) (v)
#endif

        // the segment's slabs (SEG); otherwise every slab, the bound re-read from shared memory
        const int slb = SEG ? seg * seg_len : 0;
        const int sle_seg = SEG ? min(WCX(na_), slb + seg_len) : 0;
#define SLE (SEG ? sle_seg : WCX(na_))
        for (int sl0 = slb; sl0 < SLE; sl0 += 32 / F3_SUB) {
            const int sl = sl0 + lane / F3_SUB, sub = lane % F3_SUB;
            int lo = 0, hi = -1;
            if (sl < SLE) {
                const float ac = fmaf((float)sl, WCX(da), WCX(a0));
                const float pa = ac - WCX(ha) - WCX(Sa), pb = ac + WCX(ha) - WCX(Sa);
                if (pa * WCX(sgn) > 0.f && pb * WCX(sgn) > 0.f) {
                    const float y1 = fmaf(pa, WCX(kl), WCX(So)), y2 = fmaf(pb, WCX(kl), WCX(So));
                    const float y3 = fmaf(pa, WCX(kr), WCX(So)), y4 = fmaf(pb, WCX(kr), WCX(So));
                    const float f0 = (fminf(fminf(y1, y2), fminf(y3, y4)) - WCX(o0)) * WCX(inv_do) + 0.5f;
                    const float f1 = (fmaxf(fmaxf(y1, y2), fmaxf(y3, y4)) - WCX(o0)) * WCX(inv_do) + 0.5f;
                    if (f1 >= -1.f && f0 <= (float)WCX(no_) + 1.f) {
                        lo = max((int)floorf(f0 - 1e-3f), 0);
                        hi = min((int)floorf(f1 + 1e-3f), WCX(no_) - 1);
                    }
                }
            }
            const int npass = __reduce_max_sync(0xffffffffu, (hi - lo + F3_SUB) / F3_SUB);
            for (int p = 0; p < npass; p++) {
                const int o = lo + sub + F3_SUB * p;
                bool nz = false;
                float4 eL = make_float4(0.f, 0.f, 0.f, 0.f), eG = make_float4(0.f, 0.f, 0.f, 0.f);
                int2 eR = make_int2(0, 0);
                if (o <= hi) {
                    const int i = WCX(xstep) ? sl : o, j = WCX(xstep) ? o : sl;
                    const float cx = fmaf((float)i, G.dx, G.x0) - WCX(Sx);
                    const float cy = fmaf((float)j, G.dy, G.y0) - WCX(Sy);
                    FpBase fb;
                    Footprint f;
                    bool cand = fmaf(WCX(nlx), cx, WCX(nly) * cy) + WCX(suppl) >= -WCX(tol_l) && fmaf(WCX(nrx), cx, WCX(nry) * cy) + WCX(suppr) >= -WCX(tol_r);
                    if (cand) {
                        // axial extent first: a column whose magnified extent misses the detector
                        // rows (helical views near the ends of the helix) is not queued
                        fp_base(G, WCX(cb), WCX(sb), i, j, fb);
                        fp_axial<ARC>(G, fb, WCX(zs), f.B0, f.H);
                        cand = f.B0 < (float)G.nt && fmaf(fnz, f.H, f.B0) > 0.f;
                    }
                    // PFX: the top-boundary gather (lane 31's upper row edge) is issued before the
                    // transaxial footprint so that its latency overlaps that arithmetic
                    float ih = 0.f, bg = 0.f, ft = 0.f;
                    unsigned cbq = 0u;
                    float2 qt = make_float2(0.f, 0.f);
                    if (PFX && cand) {
                        // voxel coordinate minus 1/2 at row unit u: f = (u - B0)/H - 1/2, clamped to
                        // [-1/2, nz - 1/2] as f = nz g - 1/2, g = sat(u ih + bg) in [0, 1]
                        // (ih = 1/(H nz), bg = (1/2 - B0/H)/nz): one FFMA.SAT instead of two clamps
                        const float invH = __fdividef(1.f, f.H);
                        ih = invH * rnz;
                        bg = fmaf(-f.B0, invH, 0.f) * rnz;
                        cbq = (unsigned)(j * G.nx + i) * (unsigned)pfx_stride - 0x4B400000u;
                        const float gt = __saturatef(fmaf((float)(RPL * 32), ih, bg));
                        ft = fmaf(gt, fnz, -0.5f);
                        const float rt = __fadd_rn(ft, 12582912.0f);
                        CTR_CHECK((unsigned long long)(cbq + __float_as_uint(rt)) <
                                      (unsigned long long)G.nxy * (unsigned)pfx_stride, "fwd top gather");
                        qt = __ldg(Q + (cbq + __float_as_uint(rt)));
                        if (TMA) {
                            // entries the lanes' rows reach: k(row 0) .. k(row RPL 32), monotone in the row
                            const float f0 = fmaf(__saturatef(bg), fnz, -0.5f);
                            const int kb = __float_as_int(__fadd_rn(f0, 12582912.0f)) - 0x4B400000;
                            const int kt = __float_as_int(rt) - 0x4B400000;
                            const int klo = kb & ~1, cnt = (kt + 2 - klo) & ~1;   // 16-byte aligned run
                            CTR_CHECK(cnt <= slot_entries && klo >= 0 && klo + cnt <= pfx_stride, "fwd run");
                            eR = make_int2((int)(cbq + 0x4B400000u) + klo, klo | (cnt << 16));
                        }
                    }
                    if (cand) {
                        fp_trans<ARC>(G, WCX(cb), WCX(sb), fb, f);
                        // F1 of the 4 detector columns from 5 edge evaluations
                        float T0 = trap_T(f, ((float)s0 - 0.5f) - f.sfc);
                        float Fc[F3_CPW];
#pragma unroll
                        for (int c = 0; c < F3_CPW; c++) {
                            const float T1 = trap_T(f, ((float)(s0 + c) + 0.5f) - f.sfc);
                            Fc[c] = (s0 + c < G.ns) ? T1 - T0 : 0.f;
                            T0 = T1;
                        }
                        if (Fc[0] > 0.f || Fc[1] > 0.f || Fc[2] > 0.f || Fc[3] > 0.f) {
                            nz = true;
                            const float Ls = PFX ? f.lxy * f.H : f.lxy;
                            eL = make_float4(Ls * Fc[0], Ls * Fc[1], Ls * Fc[2], Ls * Fc[3]);
                            if (PFX) {
                                eG = make_float4(ih, bg, __uint_as_float(cbq), fmaf(ft, qt.y, qt.x));
                            } else {
                                eG = make_float4(f.B0, f.H, __int_as_float(j * G.nx + i), 0.f);
                            }
                        }
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, nz);
                const int n = __popc(m);
                if (nz) {
                    const int slot = __popc(m & lanemask_lt);
                    CTR_CHECK(slot < 32, "fwd queue slot");
                    qL[wid][slot] = eL;
                    qG[wid][slot] = eG;
                    if (TMA) qR[wid][slot] = eR;
                }
                __syncwarp();
                if (TMA && lane == 0) {
                    for (int q = 0; q < min(TD, n); q++) {
                        const unsigned sl = (tcnt + q) % TD;
                        const int2 R = qR[wid][q];
                        bulk_copy(smem_u32(fwd_ring + (wid * TD + sl) * slot_entries), Q + (unsigned)R.x,
                                  (unsigned)(R.y >> 16) * 8u, smem_u32(&fbar[wid][sl]));
                    }
                }
#pragma unroll (kF3SingleUnroll)
                for (int e = 0; e < n; e++) {
                    const float4 L4 = qL[wid][e];
                    const float4 q = qG[wid][e];
                    const int col = __float_as_int(q.z);
                    float Rs[RPL];   // F2-weighted row sums of this voxel column
                    if (PFX) {
                        // X(u) = A_k + f x_k (A_k = P_k - (k - 1/2) x_k; f the voxel coordinate
                        // minus 1/2 of row boundary u, clamped to [-1/2, nz - 1/2] as f = nz g - 1/2
                        // with g = sat(u ih + bg); k = round(f) by the 1.5 2^23 magic number, either
                        // rounding of a tie giving the same X: X is continuous and Q_nz = (P_nz, 0))
                        // at the lower boundary of each of the lane's rows; the upper boundary of a
                        // row is the next row's lower one (the next lane's, by a rotation shuffle;
                        // lane 31 takes lane 0's next row, or the producer's X at the top).
                        // Unsigned 32-bit element offsets.
                        const unsigned cq = __float_as_uint(q.z);
                        float Xp[RPL];
                        const float2* __restrict__ run = nullptr;
                        int klo = 0;
                        unsigned sl = 0;
                        if (TMA) {
                            sl = (tcnt + e) % TD;
                            mbar_wait(smem_u32(&fbar[wid][sl]), ((tcnt + e) / TD) & 1);
                            klo = qR[wid][e].y & 0xffff;
                            run = fwd_ring + (wid * TD + sl) * slot_entries - klo;
                        }
#pragma unroll
                        for (int r = 0; r < RPL; r++) {
                            const float g = __saturatef(fmaf((float)fwd_row<RPL>(lane, r), q.x, q.y));
                            const float f = fmaf(g, fnz, -0.5f);
                            const float rm = __fadd_rn(f, 12582912.0f);
                            float2 qk;
                            if (TMA) {
                                const int k = __float_as_int(rm) - 0x4B400000;
                                CTR_CHECK(k >= klo && k < klo + (qR[wid][e].y >> 16), "fwd run entry");
                                qk = run[k];
                            } else {
                                CTR_CHECK((unsigned long long)(cq + __float_as_uint(rm)) <
                                              (unsigned long long)G.nxy * (unsigned)pfx_stride, "fwd prefix gather");
                                qk = __ldg(Q + (cq + __float_as_uint(rm)));
                            }
                            Xp[r] = fmaf(f, qk.y, qk.x);
                        }
                        if (TMA) {
                            // every lane has read slot sl: refill it with hit e + TD
                            __syncwarp();
                            if (lane == 0 && e + TD < n) {
                                const int2 R = qR[wid][e + TD];
                                bulk_copy(smem_u32(fwd_ring + (wid * TD + sl) * slot_entries), Q + (unsigned)R.x,
                                          (unsigned)(R.y >> 16) * 8u, smem_u32(&fbar[wid][sl]));
                            }
                        }
                        if (F3_STRIDED) {
                            float v[RPL];
#pragma unroll
                            for (int r = 0; r < RPL; r++) v[r] = __shfl_sync(0xffffffffu, Xp[r], (lane + 1) & 31);
#pragma unroll
                            for (int r = 0; r < RPL; r++)
                                Rs[r] = (lane < 31 ? v[r] : (r + 1 < RPL ? v[(r + 1) % RPL] : q.w)) - Xp[r];
                        } else {
                            const float xn = __shfl_down_sync(0xffffffffu, Xp[0], 1);
#pragma unroll
                            for (int r = 0; r < RPL; r++)
                                Rs[r] = (r + 1 < RPL ? Xp[(r + 1) % RPL] : (lane == 31 ? q.w : xn)) - Xp[r];
                        }
                    } else {
                        const float* __restrict__ xc = x + col;
                        const float btop = fmaf(fnz, q.y, q.x);
#pragma unroll
                        for (int r = 0; r < RPL; r++) {
                            const int t = fwd_row<RPL>(lane, r);
                            const float tb = (float)t, tb1 = (float)(t + 1);
                            float a = 0.f;
                            if (t < G.nt && tb1 > q.x && tb < btop) {
                                int k = (int)floorf((tb - q.x) / q.y);
                                k = min(max(k, 0), G.nz - 1);
                                while (k > 0 && fmaf((float)k, q.y, q.x) > tb) k--;
                                float bk = fmaf((float)k, q.y, q.x);
                                for (; k < G.nz; k++) {
                                    if (bk >= tb1) break;
                                    const float bk1 = fmaf((float)(k + 1), q.y, q.x);
                                    const float ov = fminf(bk1, tb1) - fmaxf(bk, tb);
                                    CTR_CHECK(k >= 0 && k < G.nz, "fwd direct z index");
                                    if (ov > 0.f) a = fmaf(ov, ONES ? 1.f : __ldg(&xc[(size_t)k * G.nxy]), a);
                                    bk = bk1;
                                }
                            }
                            Rs[r] = a;
                        }
                    }
#pragma unroll
                    for (int r = 0; r < RPL; r++) {
#if F3_CREDIT2
                        acc2[0][r] = fma2(make_float2(L4.x, L4.y), bcast2(Rs[r]), acc2[0][r]);
                        acc2[1][r] = fma2(make_float2(L4.z, L4.w), bcast2(Rs[r]), acc2[1][r]);
#else
                        acc[0][r] = fmaf(L4.x, Rs[r], acc[0][r]);
                        acc[1][r] = fmaf(L4.y, Rs[r], acc[1][r]);
                        acc[2][r] = fmaf(L4.z, Rs[r], acc[2][r]);
                        acc[3][r] = fmaf(L4.w, Rs[r], acc[3][r]);
#endif
                    }
                }
                if (TMA) tcnt += n;
                __syncwarp();
            }
        }
    }

#undef WCX
#undef SLE
    // epilogue: stage [row][detector column in block], then each thread handles one (row, column)
#pragma unroll
    for (int c = 0; c < F3_CPW; c++)
#pragma unroll
        for (int r = 0; r < RPL; r++)
#if F3_CREDIT2
            stage[fwd_row<RPL>(lane, r)][wid * F3_CPW + c] = (c & 1) ? acc2[c >> 1][r].y : acc2[c >> 1][r].x;
#else
            stage[fwd_row<RPL>(lane, r)][wid * F3_CPW + c] = acc[c][r];
#endif
#if F3_PREYW
    if (YW) asm volatile("cp.async.wait_all;" ::: "memory");
#endif
    __syncthreads();
    if (SEG) {
        // raw row sums of this segment (L_z, w and y are applied by k_fwd3_reduce)
        float* __restrict__ pp = out + (size_t)(seg * part_views + vi) * G.nt * G.ns;
        for (int q = threadIdx.x; q < G.nt * (NW * F3_CPW); q += (32 * NW)) {
            const int t = q / (NW * F3_CPW), c = q % (NW * F3_CPW);
            const int ss = sb0 + c;
            if (ss < G.ns) __stcg(pp + (size_t)t * G.ns + ss, stage[t][c]);
        }
    }
    for (int q = threadIdx.x; !SEG && q < G.nt * (NW * F3_CPW); q += (32 * NW)) {
        const int t = q / (NW * F3_CPW), c = q % (NW * F3_CPW);
        const int ss = sb0 + c;
        if (ss >= G.ns) continue;
        const float lz = ray_Lz<ARC>(G, ss, t);
        CTR_CHECK(t < 32 * RPL, "fwd stage row");
        const float p = lz * stage[t][c];
        const size_t o = ((size_t)vi * G.nt + t) * G.ns + ss;
        if (MODE == FWD_PLAIN) {
            out[o] = p;
        } else {
#if F3_PREYW
            const float wv = w ? wsm[t][c] : 1.f;
            if (MODE == FWD_RESID) out[o] = lz * wv * (p - ysm[t][c]);
            else out[o] = lz * wv * p;
#else
            // y, w are read once per sub-iteration: streaming (evict-first) loads
            const size_t a = ((size_t)v * G.nt + t) * G.ns + ss;
            const float wv = w ? __ldcs(&w[a]) : 1.f;
            if (MODE == FWD_RESID) out[o] = lz * wv * (p - __ldcs(&y[a]));
            else out[o] = lz * wv * p;
#endif
        }
    }
}

// TMA variant: entries of the longest run a hit can need — RPL 32 detector rows over the smallest
// voxel height H_min = dz Dsd / ((Dso + r_xy) dt) (the magnification of the farthest voxel) — plus
// rounding and alignment, at most a whole column
static int fwd_slot_entries(const DGeom& G, int rpl, int ps) {
    const double hmin = (double)G.dz * G.dsd / ((double)G.dso + G.rxy) * G.inv_dt;
    const int run = (int)std::ceil(32.0 * rpl / hmin) + 6;
    return std::min(ps, (run + 1) & ~1);
}

template <bool ARC, int MODE, int RPL, bool PFX, int NW>
static void fwd3_launch(const DGeom& G, dim3 grid, const float4* vtab, const Ctl* ctl, Views v, const float* xa,
                        const float* xb, const float* y, const float* w, float* out, int ps, cudaStream_t s) {
    const int se = (PFX && F3_TMA) ? fwd_slot_entries(G, RPL, ps) : 0;
    const size_t smem = (size_t)NW * F3_TMAD * se * sizeof(float2);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_fwd3<ARC, MODE, RPL, PFX, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(k_fwd3<ARC, MODE, RPL, PFX, NW>, grid, 32 * NW, smem, s, G, vtab, ctl, v, xa, xb, y, w, out, ps, se, nullptr, 0, 0);
}

template <bool ARC, int MODE, bool PFX, int NW>
static void fwd3_nw(const DGeom& G, int max_count, const float4* vtab, const Ctl* ctl, Views v, const float* xa,
                    const float* xb, const float* y, const float* w, float* out, int ps, cudaStream_t s) {
    dim3 grid((G.ns + NW * F3_CPW - 1) / (NW * F3_CPW), max_count);
    if (G.nt <= 32) fwd3_launch<ARC, MODE, 1, PFX, NW>(G, grid, vtab, ctl, v, xa, xb, y, w, out, ps, s);
    else if (G.nt <= 64) fwd3_launch<ARC, MODE, 2, PFX, NW>(G, grid, vtab, ctl, v, xa, xb, y, w, out, ps, s);
    else fwd3_launch<ARC, MODE, 4, PFX, NW>(G, grid, vtab, ctl, v, xa, xb, y, w, out, ps, s);
}

// 2-warp blocks when 4-warp blocks would fill fewer than two waves (8 blocks per SM)
template <bool ARC, int MODE, bool PFX>
static void fwd3_rpl(const DGeom& G, int max_count, const float4* vtab, const Ctl* ctl, Views v, const float* xa,
                     const float* xb, const float* y, const float* w, float* out, int ps, cudaStream_t s) {
    const long long blocks4 = (long long)((G.ns + F3_CPB - 1) / F3_CPB) * max_count;
    if (blocks4 < 148LL * F3_MINB * 2)
        fwd3_nw<ARC, MODE, PFX, F3_NWARPS / 2>(G, max_count, vtab, ctl, v, xa, xb, y, w, out, ps, s);
    else
        fwd3_nw<ARC, MODE, PFX, F3_NWARPS>(G, max_count, vtab, ctl, v, xa, xb, y, w, out, ps, s);
}

template <bool ARC>
static void fwd3_dispatch(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, int max_count,
                          const float* xa, const float* xb, const float* y, const float* w, float* out, int mode,
                          int pfx_stride, cudaStream_t s) {
    const bool pfx = pfx_stride > 0;
    if (mode == FWD_PLAIN) {
        pfx ? fwd3_rpl<ARC, FWD_PLAIN, true>(G, max_count, vtab, ctl, v, xa, xb, y, w, out, pfx_stride, s)
            : fwd3_rpl<ARC, FWD_PLAIN, false>(G, max_count, vtab, ctl, v, xa, xb, y, w, out, 0, s);
    } else if (mode == FWD_RESID) {
        pfx ? fwd3_rpl<ARC, FWD_RESID, true>(G, max_count, vtab, ctl, v, xa, xb, y, w, out, pfx_stride, s)
            : fwd3_rpl<ARC, FWD_RESID, false>(G, max_count, vtab, ctl, v, xa, xb, y, w, out, 0, s);
    } else {
        fwd3_rpl<ARC, FWD_ONES_W, false>(G, max_count, vtab, ctl, v, xa, xb, y, w, out, 0, s);
    }
}

template <bool ARC>
static void fwd2_dispatch(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, int max_count,
                          const float* xa, const float* xb, const float* y, const float* w, float* out, int mode,
                          cudaStream_t s) {
    if (F2B) {
        // the widest cell group (32, 16, 8) that still gives >= 4 blocks per SM (c2: 32, c1: 16;
        // measured, profiles/r2s/fwd2b_ab.log: wider groups evaluate each footprint fewer times)
        const long long need = 148LL * F2B_MINBPS;
        int cpb = F2B_CPB;
        if (cpb == 0) cpb = (long long)((G.ns + 31) / 32) * max_count >= need ? 32
                            : (long long)((G.ns + 15) / 16) * max_count >= need ? 16 : 8;
        if (cpb == 8) {
            dim3 grid((G.ns + 7) / 8, max_count);
            if (mode == FWD_PLAIN) launch_k(k_fwd2b<ARC, FWD_PLAIN, 8, 4>, grid, 128, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
            else if (mode == FWD_RESID) launch_k(k_fwd2b<ARC, FWD_RESID, 8, 4>, grid, 128, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
            else launch_k(k_fwd2b<ARC, FWD_ONES_W, 8, 4>, grid, 128, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
        } else if (cpb == 16) {
            dim3 grid((G.ns + 15) / 16, max_count);
            if (mode == FWD_PLAIN) launch_k(k_fwd2b<ARC, FWD_PLAIN, 16, 4>, grid, 128, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
            else if (mode == FWD_RESID) launch_k(k_fwd2b<ARC, FWD_RESID, 16, 4>, grid, 128, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
            else launch_k(k_fwd2b<ARC, FWD_ONES_W, 16, 4>, grid, 128, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
        } else {
            dim3 grid((G.ns + 31) / 32, max_count);
            if (mode == FWD_PLAIN) launch_k(k_fwd2b<ARC, FWD_PLAIN, 32, 8>, grid, 256, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
            else if (mode == FWD_RESID) launch_k(k_fwd2b<ARC, FWD_RESID, 32, 8>, grid, 256, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
            else launch_k(k_fwd2b<ARC, FWD_ONES_W, 32, 8>, grid, 256, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
        }
        return;
    }
    dim3 grid((G.ns + F2_CPW * F2_GPB - 1) / (F2_CPW * F2_GPB), max_count);
    const int bs = 32 * F2_WARPS;
    if (mode == FWD_PLAIN) launch_k(k_fwd2<ARC, FWD_PLAIN>, grid, bs, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
    else if (mode == FWD_RESID) launch_k(k_fwd2<ARC, FWD_RESID>, grid, bs, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
    else launch_k(k_fwd2<ARC, FWD_ONES_W>, grid, bs, 0, s, G, vtab, ctl, v, xa, xb, y, w, out);
}

// r / L_z(s, t): the solver's residual buffer holds L_z W (A x - y) (L_z folded in for the
// back-projector, which then needs none); oslalm_residual returns W (A x - y).
template <bool ARC>
__global__ void k_unfold_lz(DGeom G, long long n, const float* __restrict__ r, float* __restrict__ out) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(q % G.ns);
        const int t = (int)((q / G.ns) % G.nt);
        out[q] = G.dim == 3 ? r[q] / ray_Lz<ARC>(G, s, t) : r[q];
    }
}

void launch_unfold_lz(const DGeom& G, int count, const float* r, float* r_out, cudaStream_t s) {
    const long long n = (long long)count * G.nt * G.ns;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (G.arc) k_unfold_lz<true><<<blocks, 256, 0, s>>>(G, n, r, r_out);
    else k_unfold_lz<false><<<blocks, 256, 0, s>>>(G, n, r, r_out);
    launches_add(1);
}

void launch_fwd(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, int max_count, const float* xa,
                const float* xb, const float* y, const float* w, float* out, int mode, cudaStream_t s,
                int pfx_stride) {
    if (max_count <= 0) return;
    if (G.arc) {
        if (G.dim == 3) fwd3_dispatch<true>(G, vtab, ctl, v, max_count, xa, xb, y, w, out, mode, pfx_stride, s);
        else fwd2_dispatch<true>(G, vtab, ctl, v, max_count, xa, xb, y, w, out, mode, s);
    } else {
        if (G.dim == 3) fwd3_dispatch<false>(G, vtab, ctl, v, max_count, xa, xb, y, w, out, mode, pfx_stride, s);
        else fwd2_dispatch<false>(G, vtab, ctl, v, max_count, xa, xb, y, w, out, mode, s);
    }
    launches_add(1);
}


// ---------------------------------------------------------------------------
// Segmented z-prefix forward (SEG above).  The segment length is a multiple of the 32-slab pass
// so that segments split no pass; the schedule is built on the host from the view table.
#ifndef FWD_SEG_TILE_MB
#define FWD_SEG_TILE_MB 40   // z-prefix MB per schedule tile (c5: 128^2, c4: 128^2, c3: 256^2 columns; profiles/r2s/tile_ab.log)
#endif
int fwd_seg_len(const DGeom& G, int nseg) {
    const int na = std::max(G.nx, G.ny);
    const int per = (na + nseg - 1) / nseg;
    return ((per + 31) / 32) * 32;
}

// Schedule of the segmented forward for views {start + vi stride}, vi < count: every
// (vi, detector-column block, segment) once, sorted by the xy tile (serpentine order) that the
// middle ray of the block crosses at the middle of the segment, then by view -- resident blocks
// then work on one tile's voxel columns (a tile's z-prefix fits L2) across consecutive views.
std::vector<int2> fwd_seg_schedule(const DGeom& G, const std::vector<float4>& htab, Views v, int count, int nseg,
                                   int* seg_len_out) {
    const int seg_len = fwd_seg_len(G, nseg);
    const int nseg_eff = (std::max(G.nx, G.ny) + seg_len - 1) / seg_len;
    const int cpb = F3_NWARPS * F3_CPW;
    const int nbx = (G.ns + cpb - 1) / cpb;
    // tile edge (voxels): about FWD_SEG_TILE_MB of z-prefix per tile, a power of two in [16, 256]
    const double per_col = 8.0 * (double)pfx_stride_of(G);
    int T = 16;
    while (T < 256 && (double)(2 * T) * (2 * T) * per_col <= FWD_SEG_TILE_MB * 1024.0 * 1024.0) T *= 2;
    const int ntx = (G.nx + T - 1) / T, nty = (G.ny + T - 1) / T;
    struct E {
        long long key;
        int2 e;
    };
    std::vector<E> ent;
    ent.reserve((size_t)count * nbx * nseg_eff);
    for (int vi = 0; vi < count; vi++) {
        const float4 vw = htab[(size_t)v.start + (size_t)vi * v.stride];
        const double cb = vw.x, sb = vw.y;
        const double Sx = G.dso * cb, Sy = G.dso * sb;
        for (int bx = 0; bx < nbx; bx++) {
            const double sm = std::min(bx * cpb + cpb / 2, G.ns - 1);
            const double tm = (sm - G.s_c0) * G.delta;
            const double cam = G.arc ? std::cos(tm) : G.dsd, cum = G.arc ? std::sin(tm) : tm;
            const double dmx = -cam * cb - cum * sb, dmy = -cam * sb + cum * cb;
            const bool xstep = std::fabs(dmx) >= std::fabs(dmy);
            for (int sg = 0; sg < nseg_eff; sg++) {
                const int na_ = xstep ? G.nx : G.ny;
                const double slab = std::min((double)sg * seg_len + 0.5 * seg_len, (double)na_ - 0.5);
                const double a = (xstep ? G.x0 : G.y0) + slab * (xstep ? G.dx : G.dy);
                const double lam = (a - (xstep ? Sx : Sy)) / (xstep ? dmx : dmy);
                const double o = (xstep ? Sy : Sx) + lam * (xstep ? dmy : dmx);
                const double px = xstep ? a : o, py = xstep ? o : a;
                int tx = (int)std::floor((px - G.x0) / G.dx / T + 0.5 / T);
                int ty = (int)std::floor((py - G.y0) / G.dy / T + 0.5 / T);
                tx = std::min(std::max(tx, 0), ntx - 1);
                ty = std::min(std::max(ty, 0), nty - 1);
                const long long tile = (long long)ty * ntx + ((ty & 1) ? ntx - 1 - tx : tx);
                const long long key = ((tile * count + vi) * nseg_eff + sg) * nbx + bx;
                ent.push_back(E{key, make_int2(vi, bx | (sg << 16))});
            }
        }
    }
    std::stable_sort(ent.begin(), ent.end(), [](const E& p, const E& q) { return p.key < q.key; });
    std::vector<int2> out(ent.size());
    for (size_t q = 0; q < ent.size(); q++) out[q] = ent[q].e;
    *seg_len_out = seg_len;
    return out;
}

// Sum of the segments' raw row sums in segment order (deterministic) + the forward's epilogue.
template <bool ARC, int MODE>
__global__ void __launch_bounds__(256) k_fwd3_reduce(DGeom G, const Ctl* __restrict__ ctl, Views vsel,
                                                     const float* __restrict__ part, int nseg, int part_views,
                                                     const float* __restrict__ y, const float* __restrict__ w,
                                                     float* __restrict__ out) {
    pdl_enter();
    const Views V = select_views(ctl, vsel);
    const long long per = (long long)G.nt * G.ns;
    const long long n = (long long)V.count * per, pstride = (long long)part_views * per;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        float acc = __ldcs(part + q);
        for (int sg = 1; sg < nseg; sg++) acc += __ldcs(part + q + sg * pstride);
        const int ss = (int)(q % G.ns), t = (int)((q / G.ns) % G.nt);
        const long long vi = q / per;
        const float lz = ray_Lz<ARC>(G, ss, t);
        const float p = lz * acc;
        if (MODE == FWD_PLAIN) {
            out[q] = p;
        } else {
            const size_t a = ((size_t)(V.start + vi * V.stride) * G.nt + t) * G.ns + ss;
            const float wv = w ? __ldcs(&w[a]) : 1.f;
            if (MODE == FWD_RESID) out[q] = lz * wv * (p - __ldcs(&y[a]));
            else out[q] = lz * wv * p;
        }
    }
}

template <bool ARC, int RPL, int NW>
static void fwd3_seg_launch(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* pfx,
                            int ps, const int2* sched, int nsched, int seg_len, int max_count, float* part,
                            cudaStream_t s) {
    launch_k(k_fwd3<ARC, FWD_PLAIN, RPL, true, NW, true>, nsched, 32 * NW, 0, s, 
        G, vtab, ctl, v, pfx, pfx, nullptr, nullptr, part, ps, 0, sched, seg_len, max_count);
}

void launch_fwd_seg(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, int max_count, const float* pfx,
                    const float* y, const float* w, float* out, int mode, cudaStream_t s, int pfx_stride,
                    const int2* sched, int nsched, int seg_len, int nseg, float* part) {
    if (max_count <= 0) return;
    constexpr int NW = F3_NWARPS;
#define CTR_SEG(ARC)                                                                                          \
    if (G.nt <= 32) fwd3_seg_launch<ARC, 1, NW>(G, vtab, ctl, v, pfx, pfx_stride, sched, nsched, seg_len, max_count, part, s); \
    else if (G.nt <= 64) fwd3_seg_launch<ARC, 2, NW>(G, vtab, ctl, v, pfx, pfx_stride, sched, nsched, seg_len, max_count, part, s); \
    else fwd3_seg_launch<ARC, 4, NW>(G, vtab, ctl, v, pfx, pfx_stride, sched, nsched, seg_len, max_count, part, s);
    if (G.arc) {
        CTR_SEG(true)
    } else {
        CTR_SEG(false)
    }
#undef CTR_SEG
    const long long n = (long long)max_count * G.nt * G.ns;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
#define CTR_RED(ARC)                                                                                               \
    if (mode == FWD_PLAIN) launch_k(k_fwd3_reduce<ARC, FWD_PLAIN>, blocks, 256, 0, s, G, ctl, v, part, nseg, max_count, y, w, out); \
    else if (mode == FWD_RESID) launch_k(k_fwd3_reduce<ARC, FWD_RESID>, blocks, 256, 0, s, G, ctl, v, part, nseg, max_count, y, w, out); \
    else launch_k(k_fwd3_reduce<ARC, FWD_ONES_W>, blocks, 256, 0, s, G, ctl, v, part, nseg, max_count, y, w, out);
    if (G.arc) {
        CTR_RED(true)
    } else {
        CTR_RED(false)
    }
#undef CTR_RED
    launches_add(2);
}

}  // namespace ctr
