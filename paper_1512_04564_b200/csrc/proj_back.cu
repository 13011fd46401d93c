// proj_back.cu — K3 (+K5 epilogue): voxel-driven separable-footprint
// back-projection, a gather over the subset's views.
//
// 3-D (k_back3): thread = one voxel column (i, j) x a z-chunk of BK_KZ voxels
// (register accumulators); block = 32 x BK_Y columns (32 consecutive x in a
// warp, so a warp's sinogram reads hit neighbouring detector columns).  The
// kernel comment below gives the per-view steps.  2-D (k_back2): thread = one
// pixel.  Both evaluate the footprint with the functions the forward uses
// (ct_internal.cuh), so A' is the transpose of A up to rounding.
//
// Epilogues (Algorithm 1; htilde form):
//   BK_WRITE   out = scale * A'r          BK_ACCUM out += scale * A'r
//   BK_INIT    zeta = M A'r;  g = zeta; htilde = zeta         (line 1)
//   BK_UPDATE  zeta = M A'r;  g = rho/(rho+1)(alpha zeta + (1-alpha) g) + g/(rho+1);
//              htilde += alpha zeta                            (lines 6-8)
//              (Algorithm 2, Ctl.simple: htilde = zeta)
#include <cstdlib>

#include "kernels.cuh"

namespace ctr {

#ifndef BK_YDIM
#define BK_YDIM 4      // voxel-column rows per block (block = 32 x BK_Y threads)
#endif
constexpr int BK_Y = BK_YDIM;
constexpr int BK_BS = 32 * BK_Y;
constexpr int BK_RMAX3 = 28;      // rows buffered per pass in k_back3 at KZ = 16 (more rows => several passes)

// 2-D back-projection: thread = one pixel and every VS-th view of the subset
// (VS > 1 for small images, so that a 128 x 128 image still fills the GPU);
// per view one footprint and the F1-weighted sum over the <= kMaxCells cells it
// covers; the VS partial sums are added in a fixed order (deterministic).
template <bool ARC, int EPI, int VS>
__global__ void __launch_bounds__(BK_BS * VS)
k_back2(DGeom G, const float4* __restrict__ vtab, const Ctl* __restrict__ ctl, Views vsel,
        const float* __restrict__ proj, float scale, float* __restrict__ out, float* __restrict__ gbuf,
        float* __restrict__ htbuf) {
    pdl_enter();
    __shared__ float red[VS][BK_Y][32];
    const int i = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * BK_Y + threadIdx.y;
    const int part = threadIdx.z;
    const bool act = i < G.nx && j < G.ny;
    const Views V = select_views(ctl, vsel);
    float acc = 0.f;
    for (int vi = part; act && vi < V.count; vi += VS) {
        const int v = V.start + vi * V.stride;
        const float4 vw = __ldg(&vtab[v]);
        Footprint f;
        ct_footprint<ARC>(G, vw.x, vw.y, vw.z, i, j, f);
        const int slo = max((int)floorf(f.sfc + f.u0 + 0.5f), 0);
        const int shi = min((int)floorf(f.sfc + f.u3 + 0.5f), G.ns - 1);
        const float* __restrict__ pr = proj + (size_t)vi * G.ns;
        float Tprev = trap_T(f, ((float)slo - 0.5f) - f.sfc);
        float rs = 0.f;
        for (int s = slo; s <= shi; s++) {
            const float Tn = trap_T(f, ((float)s + 0.5f) - f.sfc);
            rs = fmaf(Tn - Tprev, __ldg(pr + s), rs);
            Tprev = Tn;
        }
        acc = fmaf(f.lxy, rs, acc);
    }
    if (VS > 1) {
        red[part][threadIdx.y][threadIdx.x] = acc;
        __syncthreads();
        acc = 0.f;
#pragma unroll
        for (int q = 0; q < VS; q++) acc += red[q][threadIdx.y][threadIdx.x];
    }
    // (no early returns: with BK_UPDATE every thread reaches advance_after_last_block)
    if (!act || part != 0) {
    } else if (EPI == BK_WRITE) {
        out[(size_t)j * G.nx + i] = scale * acc;
    } else if (EPI == BK_ACCUM) {
        out[(size_t)j * G.nx + i] += scale * acc;
    } else if (EPI == BK_INIT) {
        gbuf[(size_t)j * G.nx + i] = scale * acc;
        htbuf[(size_t)j * G.nx + i] = scale * acc;
    } else {
        const size_t idx = (size_t)j * G.nx + i;
        const float z = scale * acc;
        const float rho = rho_of_k(ctl), alpha = ctl->alpha;
        const float gv = gbuf[idx];
        const float inv = 1.f / (rho + 1.f);
        gbuf[idx] = fmaf(rho * inv, fmaf(alpha, z, (1.f - alpha) * gv), gv * inv);
        htbuf[idx] = ctl->simple ? z : fmaf(alpha, z, htbuf[idx]);
    }
    if (EPI == BK_UPDATE) advance_after_last_block(ctl);
}

// Row sums of one (voxel column, view) over a window of W detector columns:
// rs(t) = sum_q F[q] r[t][sw + q] (L_z(s, t) folded in when LZ), stored with
// the running sum in affine form, cs[o] = (C_o - (o - 1/2) rs(t), rs(t)) with
// C_o = sum_{t' < t} rs and o = t - tw, so that the cumulative at row
// coordinate v in [o - 1/2, o + 1/2] is one FFMA, cs[o].x + v cs[o].y.  The next row's W
// gathers are issued before the current row's FMAs (software pipelining).
#ifndef BK_WMAX
#define BK_WMAX 6      // widest register window of detector columns (wider footprints: general loop)
#endif

// BK_PEEL: the row loop prefetches row o + 1 unconditionally and the last row is peeled (no
// per-row select of the prefetch address: 62 instead of 67 instructions per 4 rows at W = 4).
// Measured slower (c4 back 2.386 vs 2.247 ms, c3 0.298 vs 0.272, c5 14.10 vs 12.98;
// profiles/r2fb/peel_ab.log): a switch only.
#ifndef BK_PEEL
#define BK_PEEL 0
#endif
// BK_PF2 = u > 0: the row loop requests row o + 2 while row o is summed (unrolled by u).
#ifndef BK_PF2
#define BK_PF2 0
#endif
// BK_RU: unroll factor of the row loop (4 = what the compiler picks on its own: the loads of four
// rows are issued together).
#ifndef BK_RU
#define BK_RU 4
#endif
template <bool ARC, bool LZ, int W>
__device__ __forceinline__ void back_rows(const DGeom& G, const float (&F)[BK_WMAX], const float* __restrict__ pr,
                                          int sw, int tw, int n, float2* __restrict__ cs, float& run) {
    float a[W], b[W];
    float ofs = 0.5f;   // 1/2 - o
#pragma unroll
    for (int q = 0; q < W; q++) a[q] = __ldg(pr + q);
    auto row = [&](int o) {
        float rs = 0.f;
#pragma unroll
        for (int q = 0; q < W; q++) {
            const float wq = LZ ? F[q] * ray_Lz<ARC>(G, sw + q, tw + o) : F[q];
            rs = fmaf(wq, a[q], rs);
        }
        CTR_CHECK(o < n, "back row buffer");
        cs[o * BK_BS] = make_float2(fmaf(ofs, rs, run), rs);
        run += rs;
        ofs -= 1.f;
    };
#if BK_PF2
    // two rows ahead: row o + 2 is requested while row o is summed (c -> b -> a)
    float c[W];
    const int ns = G.ns;
    {
        const float* __restrict__ p1 = pr + (1 < n ? ns : 0);
#pragma unroll
        for (int q = 0; q < W; q++) b[q] = __ldg(p1 + q);
        pr = p1;
    }
    constexpr int PFU = BK_PF2;
#pragma unroll PFU
    for (int o = 0; o < n; o++) {
        const float* __restrict__ pn = pr + (o + 2 < n ? ns : 0);
#pragma unroll
        for (int q = 0; q < W; q++) c[q] = __ldg(pn + q);
        row(o);
        pr = pn;
#pragma unroll
        for (int q = 0; q < W; q++) {
            a[q] = b[q];
            b[q] = c[q];
        }
    }
#elif BK_PEEL
    for (int o = 0; o < n - 1; o++) {
        pr += G.ns;
#pragma unroll
        for (int q = 0; q < W; q++) b[q] = __ldg(pr + q);
        row(o);
#pragma unroll
        for (int q = 0; q < W; q++) a[q] = b[q];
    }
    row(n - 1);
#else
    constexpr int RU = BK_RU;
#pragma unroll RU
    for (int o = 0; o < n; o++) {
        const float* __restrict__ pn = pr + (o + 1 < n ? G.ns : 0);
#pragma unroll
        for (int q = 0; q < W; q++) b[q] = __ldg(pn + q);
        row(o);
        pr = pn;
#pragma unroll
        for (int q = 0; q < W; q++) a[q] = b[q];
    }
#endif
}

// ---------------------------------------------------------------------------
// 3-D back-projection.  Thread = one voxel column (i, j) x a z-chunk of BK_KZ
// voxels; block = 32 x BK_Y columns.  Per view:
//   1. axial extent first (fp_base + fp_axial: ~20 instructions): a chunk
//      whose rows [B0 + k0 H, B0 + (k0+kz) H] miss the detector skips the view
//      (helical views see a z-band only);
//   2. transaxial footprint (fp_trans) and F1 of the <= 4 detector columns it
//      covers, kept in registers (wider footprints take a general loop);
//   3. per row t: rs(t) = L_xy sum_s F1(s) r[t][s] (4 gathers + 4 FMA), stored
//      with its running sum as float2 (cs_t, rs_t) in a per-thread
//      shared-memory column;
//   4. per voxel: the F2-weighted row sum is R(b_k+1) - R(b_k) with the
//      piecewise-linear cumulative R(u) = A_o + v rs_o, A_o = cs_o - (o - 1/2) rs_o
//      (one 8-byte shared load and one FFMA per voxel boundary, magic-number
//      rounding).
template <bool ARC, int EPI, bool LZ, int BK_KZ>
#ifndef BK_VSM
#define BK_VSM 128     // view descriptors of the block's window staged in shared memory
#endif
#ifndef BK_EPB
#define BK_EPB 12      // voxels per batch of the g/htilde epilogue (loads of a batch issued together)
#endif
#ifndef BK_RM24
#define BK_RM24 40     // rows buffered per pass at KZ = 24 (41 x 128 float2 = 42 KB)
#endif
#ifndef BK_MINB24
#define BK_MINB24 5    // resident blocks per SM at KZ = 24 (<= 102 registers)
#endif
__global__ void __launch_bounds__(BK_BS, BK_KZ <= 16 ? 7 : BK_KZ <= 24 ? BK_MINB24 : 3)
k_back3(DGeom G, const float4* __restrict__ vtab, const Ctl* __restrict__ ctl, Views vsel,
        const float* __restrict__ proj, float scale, float* __restrict__ out, float* __restrict__ gbuf,
        float* __restrict__ htbuf) {
    pdl_enter();
    constexpr int RM = BK_KZ <= 8 ? 14 : BK_KZ <= 16 ? BK_RMAX3 : BK_KZ <= 24 ? BK_RM24 : 44;
    __shared__ float2 csb[RM + 1][BK_BS];
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int i = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * BK_Y + threadIdx.y;
    const int k0 = blockIdx.z * BK_KZ;
    const Views V = select_views(ctl, vsel);
    const int nt = G.nt;
    const float fkz = (float)min(BK_KZ, G.nz - k0);

    // Helical view window of the block's z-chunk: the chunk [zlo, zhi] can reach the
    // detector rows [0, nt) only if zlo - (nt - tc)/m < z_s < zhi + tc/m for some
    // magnification m in [Dsd / (dso + rxy), Dsd / (dso - rxy)] / dt (row units, tc the
    // row of z = z_s), so views whose source z is outside that window (plus a 1 mm /
    // 1 view margin) are skipped for the whole block before the per-column test below.
    int vi0 = 0, vi1 = V.count;
    if (G.zstep != 0.f && V.count > 0) {
        const float mlo = G.dsd / (G.dso + G.rxy) * G.inv_dt, mhi = G.dsd / (G.dso - G.rxy) * G.inv_dt;
        const float zlo = G.zbot + (float)k0 * G.dz, zhi = zlo + fkz * G.dz;
        const float up = (float)nt - G.t_c0p;   // rows above / below the row of z = z_s
        const float wlo = zlo - fmaxf(up / mlo, up / mhi) - 1.f;
        const float whi = zhi + fmaxf(G.t_c0p / mlo, G.t_c0p / mhi) + 1.f;
        // z_s(v_i) = zs0 + (start + i stride) zstep, monotone in i
        const float a = G.zs0 + (float)V.start * G.zstep, b = (float)V.stride * G.zstep;
        float ia = (wlo - a) / b, ib = (whi - a) / b;
        if (ia > ib) { const float t = ia; ia = ib; ib = t; }
        vi0 = max(vi0, (int)floorf(ia) - 1);
        vi1 = min(vi1, (int)ceilf(ib) + 2);
    }
    // the window's view descriptors in shared memory (the per-view set-up otherwise waits on a
    // global load the row gathers have evicted from L1); views past BK_VSM are read directly
    __shared__ float4 vsm[BK_VSM];
    const int nstage = max(0, min(vi1 - vi0, BK_VSM));
    for (int q = tid; q < nstage; q += BK_BS) vsm[q] = __ldg(&vtab[V.start + (vi0 + q) * V.stride]);
    __syncthreads();
    const bool act3 = i < G.nx && j < G.ny;
    if (!act3) {
        if (EPI != BK_UPDATE) return;
        vi1 = vi0;   // BK_UPDATE: no views, no epilogue, but the block's completion is counted
    }
    float2* __restrict__ cs = &csb[0][tid];

    float acc[BK_KZ];
#pragma unroll
    for (int q = 0; q < BK_KZ; q++) acc[q] = 0.f;

    for (int vi = vi0; vi < vi1; vi++) {
        const float4 vw = vi - vi0 < BK_VSM ? vsm[vi - vi0] : __ldg(&vtab[V.start + vi * V.stride]);
        FpBase fb;
        fp_base(G, vw.x, vw.y, i, j, fb);
        float B0, H;
        fp_axial<ARC>(G, fb, vw.z, B0, H);
        const float clo = fmaf((float)k0, H, B0);
        const float chi = fmaf(fkz, H, clo);
        const int t0 = max((int)floorf(clo), 0);
        const int t1 = min((int)ceilf(chi), nt) - 1;
        if (t0 > t1) continue;
        Footprint f;
        fp_trans<ARC>(G, vw.x, vw.y, fb, f);
        // detector columns under the footprint
        const int slo = max((int)floorf(f.sfc + f.u0 + 0.5f), 0);
        const int shi = min((int)floorf(f.sfc + f.u3 + 0.5f), G.ns - 1);
        const int nc = shi - slo + 1;
        if (nc <= 0) continue;
        const unsigned pv = (unsigned)(vi * nt) * (unsigned)G.ns;  // < 2^32 (checked at launch)
        // warp-uniform window of W = 4 or BK_WMAX detector columns [sw, sw + W - 1] inside the
        // detector (F1 is exactly 0 outside [u0, u3]); wider footprints take a general loop
        const int ncmax = __reduce_max_sync(__activemask(), nc);
        const int W = (ncmax <= 4 && G.ns >= 4) ? 4 : (ncmax <= BK_WMAX && G.ns >= BK_WMAX) ? BK_WMAX : 0;
        const int sw = W ? max(min(slo, G.ns - W), 0) : slo;
        float F[BK_WMAX];
        {
            float Tprev = trap_T(f, ((float)sw - 0.5f) - f.sfc);
#pragma unroll
            for (int q = 0; q < BK_WMAX; q++) {
                if (q < 4 || q < W) {
                    const float Tn = trap_T(f, ((float)(sw + q) + 0.5f) - f.sfc);
                    F[q] = (Tn - Tprev) * f.lxy;
                    Tprev = Tn;
                } else {
                    F[q] = 0.f;
                }
            }
        }
        const float Bs = B0 - 0.5f;  // voxel boundary in row units minus (row + 1/2) below
        for (int tw = t0; tw <= t1; tw += RM) {
            const int twe = min(t1, tw + RM - 1);
            const int n = twe - tw + 1;
            CTR_CHECK(n >= 1 && n <= RM, "back rows per pass");
            float run = 0.f;
            const float* __restrict__ pr = proj + (pv + (unsigned)tw * (unsigned)G.ns + (unsigned)sw);
            if (W == 4) {
                back_rows<ARC, LZ, 4>(G, F, pr, sw, tw, n, cs, run);
            } else if (W == BK_WMAX) {
                back_rows<ARC, LZ, BK_WMAX>(G, F, pr, sw, tw, n, cs, run);
            } else {
                // wide footprint (near the source in steep geometries): F1 on the fly
                for (int o = 0; o < n; o++) {
                    const int t = tw + o;
                    float rs = 0.f;
                    float Tprev = trap_T(f, ((float)slo - 0.5f) - f.sfc);
                    for (int q = 0; q < nc; q++) {
                        const float Tn = trap_T(f, ((float)(slo + q) + 0.5f) - f.sfc);
                        const float wq = LZ ? (Tn - Tprev) * f.lxy * ray_Lz<ARC>(G, slo + q, t) : (Tn - Tprev) * f.lxy;
                        rs = fmaf(wq, __ldg(pr + q), rs);
                        Tprev = Tn;
                    }
                    cs[o * BK_BS] = make_float2(fmaf(0.5f - (float)o, rs, run), rs);
                    run += rs;
                    pr += G.ns;
                }
            }
            cs[n * BK_BS] = make_float2(run, 0.f);
            // R(u) at voxel boundary u = B0 + k H: v = u - (tw + 1/2) clamped to [-1/2, n - 1/2],
            // o = round(v) (magic number), R = cs[o].x + v cs[o].y (affine form above;
            // cs[n] = (C_n, 0)).  The clamp is a saturation: v = n g - 1/2 with
            // g = sat((q H + base + 1/2)/n) (FFMA.SAT; q is a compile-time constant after
            // unrolling); v and o of two boundaries at a time in packed FP32 (FFMA2, FADD2), and
            // the two voxels' increments R(q+1) - R(q) added with one FADD2.
            const float base = fmaf((float)k0, H, Bs - (float)tw);
            const float fn = (float)n, rn = __fdividef(1.f, fn);
            const float Hn = H * rn, bn = (base + 0.5f) * rn;
            auto R2 = [&](int q) {   // boundaries q, q + 1
                const float2 gg = make_float2(__saturatef(fmaf((float)q, Hn, bn)),
                                              __saturatef(fmaf((float)(q + 1), Hn, bn)));
                const float2 vv = fma2(gg, bcast2(fn), bcast2(-0.5f));
                const float2 rm = add2(vv, bcast2(12582912.0f));
                CTR_CHECK(__float_as_int(rm.x) - 0x4B400000 >= 0 && __float_as_int(rm.x) - 0x4B400000 <= n &&
                              __float_as_int(rm.y) - 0x4B400000 >= 0 && __float_as_int(rm.y) - 0x4B400000 <= n,
                          "back boundary row");
                const float2 ca = cs[(__float_as_int(rm.x) - 0x4B400000) * BK_BS];
                const float2 cb = cs[(__float_as_int(rm.y) - 0x4B400000) * BK_BS];
                return make_float2(fmaf(vv.x, ca.y, ca.x), fmaf(vv.y, cb.y, cb.x));
            };
            float Rlo;
            {
                const float g0 = __saturatef(bn);
                const float v0 = fmaf(g0, fn, -0.5f);
                const float2 c0 = cs[(__float_as_int(__fadd_rn(v0, 12582912.0f)) - 0x4B400000) * BK_BS];
                Rlo = fmaf(v0, c0.y, c0.x);
            }
            static_assert(BK_KZ % 2 == 0, "voxel pairs");
#pragma unroll
            for (int q = 0; q < BK_KZ; q += 2) {
                const float2 Rh = R2(q + 1);
                const float2 a2 = add2(make_float2(acc[q], acc[q + 1]), make_float2(Rh.x - Rlo, Rh.y - Rh.x));
                acc[q] = a2.x;
                acc[q + 1] = a2.y;
                Rlo = Rh.y;
            }
        }
    }

    // epilogue
    const int kz = act3 ? min(BK_KZ, G.nz - k0) : 0;
    if (EPI == BK_UPDATE) {
        // lines 7-8: g and htilde of the chunk in batches of EB voxels, every load of a batch
        // issued before its first use (one HBM round trip per batch instead of per voxel)
        const float rho = rho_of_k(ctl), alpha = ctl->alpha;
        const bool simple = ctl->simple;
        const float inv = 1.f / (rho + 1.f), ri = rho * inv, oma = 1.f - alpha;
        const size_t base = (size_t)k0 * G.nxy + (size_t)j * G.nx + i;
        constexpr int EB = (BK_KZ % BK_EPB == 0) ? BK_EPB : 8;
#pragma unroll
        for (int b = 0; b < BK_KZ; b += EB) {
            float gv[EB], hv[EB];
#pragma unroll
            for (int q = 0; q < EB; q++) {
                gv[q] = hv[q] = 0.f;
                if (b + q < kz) {
                    const size_t idx = base + (size_t)(b + q) * G.nxy;
                    gv[q] = gbuf[idx];
                    if (!simple) hv[q] = htbuf[idx];
                }
            }
#pragma unroll
            for (int q = 0; q < EB; q++) {
                if (b + q < kz) {
                    const size_t idx = base + (size_t)(b + q) * G.nxy;
                    const float z = scale * acc[b + q];
                    gbuf[idx] = fmaf(ri, fmaf(alpha, z, oma * gv[q]), gv[q] * inv);
                    htbuf[idx] = simple ? z : fmaf(alpha, z, hv[q]);
                }
            }
        }
        advance_after_last_block(ctl);
    } else {
#pragma unroll
        for (int q = 0; q < BK_KZ; q++) {
            if (q < kz) {
                const size_t idx = (size_t)(k0 + q) * G.nxy + (size_t)j * G.nx + i;
                const float z = scale * acc[q];
                if (EPI == BK_WRITE) {
                    out[idx] = z;
                } else if (EPI == BK_ACCUM) {
                    out[idx] += z;
                } else {
                    gbuf[idx] = z;
                    htbuf[idx] = z;
                }
            }
        }
    }
}

template <bool ARC, int KZ>
static void back3_dispatch_kz(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* proj,
                              float scale, int epi, bool lz, float* out, float* g, float* ht, cudaStream_t s) {
    dim3 block(32, BK_Y);
    dim3 grid((G.nx + 31) / 32, (G.ny + BK_Y - 1) / BK_Y, (G.nz + KZ - 1) / KZ);
    switch (epi) {
        case BK_WRITE:
            if (lz) launch_k(k_back3<ARC, BK_WRITE, true, KZ>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht);
            else launch_k(k_back3<ARC, BK_WRITE, false, KZ>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
        case BK_ACCUM:
            if (lz) launch_k(k_back3<ARC, BK_ACCUM, true, KZ>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht);
            else launch_k(k_back3<ARC, BK_ACCUM, false, KZ>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
        case BK_INIT:
            launch_k(k_back3<ARC, BK_INIT, false, KZ>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
        default:
            launch_k(k_back3<ARC, BK_UPDATE, false, KZ>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
    }
}

template <bool ARC>
static void back2_dispatch(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* proj,
                           float scale, int epi, float* out, float* g, float* ht, cudaStream_t s) {
    dim3 grid((G.nx + 31) / 32, (G.ny + BK_Y - 1) / BK_Y, 1);
    // split the views over 4 threads per pixel when the image has fewer blocks than ~4 per SM
    if ((long long)grid.x * grid.y < 148LL * 4) {
        dim3 block(32, BK_Y, 4);
        switch (epi) {
            case BK_WRITE: launch_k(k_back2<ARC, BK_WRITE, 4>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
            case BK_ACCUM: launch_k(k_back2<ARC, BK_ACCUM, 4>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
            case BK_INIT: launch_k(k_back2<ARC, BK_INIT, 4>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
            default: launch_k(k_back2<ARC, BK_UPDATE, 4>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
        }
        return;
    }
    // fewer than ~16 blocks per SM: two threads per pixel (the last partial wave otherwise idles SMs)
    if ((long long)grid.x * grid.y < 148LL * 16) {
        dim3 block(32, BK_Y, 2);
        switch (epi) {
            case BK_WRITE: launch_k(k_back2<ARC, BK_WRITE, 2>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
            case BK_ACCUM: launch_k(k_back2<ARC, BK_ACCUM, 2>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
            case BK_INIT: launch_k(k_back2<ARC, BK_INIT, 2>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
            default: launch_k(k_back2<ARC, BK_UPDATE, 2>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
        }
        return;
    }
    dim3 block(32, BK_Y, 1);
    switch (epi) {
        case BK_WRITE: launch_k(k_back2<ARC, BK_WRITE, 1>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
        case BK_ACCUM: launch_k(k_back2<ARC, BK_ACCUM, 1>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
        case BK_INIT: launch_k(k_back2<ARC, BK_INIT, 1>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
        default: launch_k(k_back2<ARC, BK_UPDATE, 1>, grid, block, 0, s, G, vtab, ctl, v, proj, scale, out, g, ht); break;
    }
}

#ifndef BK_KZSEL
#define BK_KZSEL 24    // voxels per thread in z (tuning variants: -DBK_KZSEL=8 | 16 | 32)
#endif
// A variant with blocks of 4 z-chunks of the same 32 columns sharing each (column, view)
// footprint through shared memory (one warp per view computes it, a barrier pair per 4 views) was
// correct but 1.7x slower (c4 4.03 vs 2.33 ms; code in commit eb51f47).

template <bool ARC, int DIM>
static void back_dispatch(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* proj,
                          float scale, int epi, bool lz, float* out, float* g, float* ht, cudaStream_t s) {
    if (DIM != 3) return back2_dispatch<ARC>(G, vtab, ctl, v, proj, scale, epi, out, g, ht, s);
    static_assert(BK_KZSEL == 8 || BK_KZSEL == 16 || BK_KZSEL == 24 || BK_KZSEL == 32, "BK_KZSEL");
    back3_dispatch_kz<ARC, BK_KZSEL>(G, vtab, ctl, v, proj, scale, epi, lz, out, g, ht, s);
}

void launch_back(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* proj, float scale,
                 int epi, bool apply_lz, float* out, float* g, float* ht, cudaStream_t s) {
    if (G.arc) {
        if (G.dim == 3) back_dispatch<true, 3>(G, vtab, ctl, v, proj, scale, epi, apply_lz, out, g, ht, s);
        else back_dispatch<true, 2>(G, vtab, ctl, v, proj, scale, epi, false, out, g, ht, s);
    } else {
        if (G.dim == 3) back_dispatch<false, 3>(G, vtab, ctl, v, proj, scale, epi, apply_lz, out, g, ht, s);
        else back_dispatch<false, 2>(G, vtab, ctl, v, proj, scale, epi, false, out, g, ht, s);
    }
    launches_add(1);
}

}  // namespace ctr

// ---------------------------------------------------------------------------
// Nonzero count of A on a set of views (the denominator of the projector's
// algorithmic FLOP figure, 2 FLOP per nonzero): entry
// ((v,t,s),(i,j,k)) is nonzero iff F1(s) > 0 and F2(k,t) > 0.
namespace ctr {

// WORK: also count[1] += in-cone voxel-view pairs (voxels with a nonzero in the
// view) and count[2] += column-view pairs with a nonzero -- the units of SURVEY
// §8d's algorithmic FLOP figure.
template <bool ARC, int DIM, bool WORK>
__global__ void __launch_bounds__(128) k_count(DGeom G, const float4* __restrict__ vtab, Views V,
                                               unsigned long long* __restrict__ count) {
    const int i = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * 4 + threadIdx.y;
    unsigned long long acc = 0, pvox = 0, pcol = 0;
    if (i < G.nx && j < G.ny) {
        for (int vi = 0; vi < V.count; vi++) {
            const float4 vw = __ldg(&vtab[V.start + vi * V.stride]);
            Footprint f;
            ct_footprint<ARC>(G, vw.x, vw.y, vw.z, i, j, f);
            const int slo = max((int)floorf(f.sfc + f.u0 + 0.5f) - 1, 0);
            const int shi = min((int)floorf(f.sfc + f.u3 + 0.5f) + 1, G.ns - 1);
            int ncz = 0;
            for (int s = slo; s <= shi; s++) ncz += sf_F1(f, s) > 0.f;
            if (ncz == 0) continue;
            long long rows = 1, vin = 1;
            if (DIM == 3) {
                rows = 0;
                vin = 0;
                for (int k = 0; k < G.nz; k++) {
                    const float lo = fmaxf(voxel_b(f, k), 0.f), hi = fminf(voxel_b(f, k + 1), (float)G.nt);
                    if (hi > lo) {
                        rows += (long long)ceilf(hi) - (long long)floorf(lo);
                        vin++;
                    }
                }
            }
            acc += (unsigned long long)ncz * (unsigned long long)rows;
            if (WORK && vin > 0) {
                pvox += (unsigned long long)vin;
                pcol++;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (WORK) {
            pvox += __shfl_down_sync(0xffffffffu, pvox, o);
            pcol += __shfl_down_sync(0xffffffffu, pcol, o);
        }
    }
    if ((threadIdx.x & 31) == 0) {
        if (acc) atomicAdd(count, acc);
        if (WORK && pvox) atomicAdd(count + 1, pvox);
        if (WORK && pcol) atomicAdd(count + 2, pcol);
    }
}

template <bool WORK>
static void count_launch(const DGeom& G, const float4* vtab, Views v, unsigned long long* count, cudaStream_t s) {
    dim3 block(32, 4), grid((G.nx + 31) / 32, (G.ny + 3) / 4);
    if (G.arc) {
        if (G.dim == 3) k_count<true, 3, WORK><<<grid, block, 0, s>>>(G, vtab, v, count);
        else k_count<true, 2, WORK><<<grid, block, 0, s>>>(G, vtab, v, count);
    } else {
        if (G.dim == 3) k_count<false, 3, WORK><<<grid, block, 0, s>>>(G, vtab, v, count);
        else k_count<false, 2, WORK><<<grid, block, 0, s>>>(G, vtab, v, count);
    }
    launches_add(1);
}

void launch_count(const DGeom& G, const float4* vtab, Views v, unsigned long long* count, cudaStream_t s) {
    count_launch<false>(G, vtab, v, count, s);
}

void launch_count_work(const DGeom& G, const float4* vtab, Views v, unsigned long long* count3, cudaStream_t s) {
    count_launch<true>(G, vtab, v, count3, s);
}

}  // namespace ctr
