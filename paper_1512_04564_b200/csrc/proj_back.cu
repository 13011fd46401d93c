// proj_back.cu — K3 (+K5 epilogue): voxel-driven separable-footprint
// back-projection, a gather over the subset's views.
//
// Thread = one voxel column (i, j) and a z-chunk of BK_KZ voxels (register
// accumulators); block = 32 x BK_Y columns (32 consecutive x in a warp, so a
// warp's sinogram reads hit consecutive detector columns).  Per view the
// thread evaluates the column's footprint once (ct_footprint, shared with the
// forward kernel), keeps F1 of its <= kMaxCells columns in a per-thread
// shared-memory slot, forms the row sums rs(t) = L_xy sum_s F1(s) r[t][s] of
// the rows its chunk projects to, then distributes them to its voxels with
// the exact overlaps F2, evaluated as differences of the cumulative row sum
// at the voxel boundaries b_k = B0 + k H (one interpolation per voxel).
//
// Epilogues (Algorithm 1; htilde form):
//   BK_WRITE   out = scale * A'r          BK_ACCUM out += scale * A'r
//   BK_INIT    zeta = M A'r;  g = zeta; htilde = zeta         (line 1)
//   BK_UPDATE  zeta = M A'r;  g = rho/(rho+1)(alpha zeta + (1-alpha) g) + g/(rho+1);
//              htilde += alpha zeta                            (lines 6-8)
#include <cstdlib>

#include "kernels.cuh"

namespace ctr {

constexpr int BK_Y = 4;
constexpr int BK_BS = 32 * BK_Y;
constexpr int BK_KZ_DEFAULT = 16;  // voxels per thread in z (tuning knob CTR_BK_KZ = 16 | 24 | 32)
constexpr int BK_RMAX = 40;  // rows buffered per pass (more rows => several passes)

template <bool ARC, int DIM, int EPI, bool LZ, int BK_KZ>
__global__ void __launch_bounds__(BK_BS)
k_back(DGeom G, const float4* __restrict__ vtab, const Ctl* __restrict__ ctl, Views vsel,
       const float* __restrict__ proj, float scale, float* __restrict__ out, float* __restrict__ gbuf,
       float* __restrict__ htbuf) {
    __shared__ float f1s[kMaxCells][BK_BS];
    __shared__ float csb[(DIM == 3) ? BK_RMAX + 2 : 1][BK_BS];
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int i = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * BK_Y + threadIdx.y;
    const int k0 = blockIdx.z * BK_KZ;
    if (i >= G.nx || j >= G.ny) return;
    const Views V = select_views(ctl, vsel);
    const int nt = (DIM == 3) ? G.nt : 1;
    const int kz = (DIM == 3) ? min(BK_KZ, G.nz - k0) : 1;

    float acc[BK_KZ];
#pragma unroll
    for (int q = 0; q < BK_KZ; q++) acc[q] = 0.f;

    for (int vi = 0; vi < V.count; vi++) {
        const int v = V.start + vi * V.stride;
        const float4 vw = __ldg(&vtab[v]);
        Footprint f;
        ct_footprint<ARC>(G, vw.x, vw.y, vw.z, i, j, f);
        int t0 = 0, t1 = 0;
        if (DIM == 3) {
            const float clo = voxel_b(f, k0), chi = voxel_b(f, k0 + kz);
            t0 = max((int)floorf(clo), 0);
            t1 = min((int)ceilf(chi), nt) - 1;
            if (t0 > t1) continue;
        }
        // detector columns under the footprint
        int slo = (int)floorf(f.sfc + f.u0 + 0.5f);
        int shi = (int)floorf(f.sfc + f.u3 + 0.5f);
        slo = max(slo, 0);
        shi = min(shi, G.ns - 1);
        int nc = shi - slo + 1;
        if (nc <= 0) continue;
        if (nc > kMaxCells) nc = kMaxCells;  // excluded at ct_geom_create (footprint bound)
        {
            float Tprev = trap_T(f, ((float)slo - 0.5f) - f.sfc);
            for (int q = 0; q < nc; q++) {
                const float Tn = trap_T(f, ((float)(slo + q) + 0.5f) - f.sfc);
                f1s[q][tid] = (Tn - Tprev) * f.lxy;
                Tprev = Tn;
            }
        }
        const unsigned pv = (unsigned)(vi * nt) * (unsigned)G.ns + (unsigned)slo;  // < 2^32 (checked at launch)
        if (DIM != 3) {
            float rs = 0.f;
            for (int q = 0; q < nc; q++) rs = fmaf(f1s[q][tid], __ldg(proj + (pv + q)), rs);
            acc[0] += rs;
            continue;
        }
        for (int tw = t0; tw <= t1; tw += BK_RMAX) {
            const int twe = min(t1, tw + BK_RMAX - 1);
            // row sums rs(t) -> running sums cs[o] = sum_{tw <= t < tw+o} rs(t) (cs[n+1] = cs[n]
            // pads the top).  The F2-weighted sum over the rows of voxel k is R(b_k+1) - R(b_k)
            // with the piecewise-linear cumulative R(u) = cs[o] + frac (cs[o+1] - cs[o]).
            const int n = twe - tw + 1;
            float run = 0.f;
            csb[0][tid] = 0.f;
            for (int t = tw; t <= twe; t++) {
                const float* __restrict__ pr = proj + (pv + (unsigned)t * (unsigned)G.ns);
                float rs = 0.f;
                if (LZ) {
                    for (int q = 0; q < nc; q++) rs = fmaf(f1s[q][tid] * ray_Lz<ARC>(G, slo + q, t), __ldg(&pr[q]), rs);
                } else {
                    for (int q = 0; q < nc; q++) rs = fmaf(f1s[q][tid], __ldg(&pr[q]), rs);
                }
                run += rs;
                csb[t - tw + 1][tid] = run;
            }
            csb[n + 1][tid] = run;
            const float shift = (float)tw + 0.5f, vmax = (float)n - 0.5f;
            auto R = [&](float u) {
                // o = round(v - 1/2), v = u - tw in [0, n]: o <= v <= o + 1 (magic-number floor)
                const float vv = fminf(fmaxf(u - shift, -0.5f), vmax);
                const float rm = __fadd_rn(vv, 12582912.0f);
                const int o = __float_as_int(rm) - 0x4B400000;
                const float fr = (vv + 0.5f) - (rm - 12582912.0f);
                const float c0 = csb[o][tid];
                return fmaf(fr, csb[o + 1][tid] - c0, c0);
            };
            float Rlo = R(voxel_b(f, k0));
#pragma unroll
            for (int q = 0; q < BK_KZ; q++) {
                if (q < kz) {
                    const float Rhi = R(voxel_b(f, k0 + q + 1));
                    acc[q] += Rhi - Rlo;
                    Rlo = Rhi;
                }
            }
        }
    }

    // epilogue
    float rho = 0.f, alpha = 0.f;
    if (EPI == BK_UPDATE) {
        rho = rho_of_k(ctl);
        alpha = ctl->alpha;
    }
#pragma unroll
    for (int q = 0; q < BK_KZ; q++) {
        if (q < kz) {
            const size_t idx = (size_t)(k0 + q) * G.nxy + (size_t)j * G.nx + i;
            const float z = scale * acc[q];
            if (EPI == BK_WRITE) {
                out[idx] = z;
            } else if (EPI == BK_ACCUM) {
                out[idx] += z;
            } else if (EPI == BK_INIT) {
                gbuf[idx] = z;
                htbuf[idx] = z;
            } else {
                const float gv = gbuf[idx];
                const float inv = 1.f / (rho + 1.f);
                gbuf[idx] = fmaf(rho * inv, fmaf(alpha, z, (1.f - alpha) * gv), gv * inv);
                htbuf[idx] = fmaf(alpha, z, htbuf[idx]);
            }
        }
    }
}

template <bool ARC, int DIM, int KZ>
static void back_dispatch_kz(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* proj,
                             float scale, int epi, bool lz, float* out, float* g, float* ht, cudaStream_t s) {
    dim3 block(32, BK_Y);
    dim3 grid((G.nx + 31) / 32, (G.ny + BK_Y - 1) / BK_Y, DIM == 3 ? (G.nz + KZ - 1) / KZ : 1);
    switch (epi) {
        case BK_WRITE:
            if (lz) k_back<ARC, DIM, BK_WRITE, true, KZ><<<grid, block, 0, s>>>(G, vtab, ctl, v, proj, scale, out, g, ht);
            else k_back<ARC, DIM, BK_WRITE, false, KZ><<<grid, block, 0, s>>>(G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
        case BK_ACCUM:
            if (lz) k_back<ARC, DIM, BK_ACCUM, true, KZ><<<grid, block, 0, s>>>(G, vtab, ctl, v, proj, scale, out, g, ht);
            else k_back<ARC, DIM, BK_ACCUM, false, KZ><<<grid, block, 0, s>>>(G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
        case BK_INIT:
            k_back<ARC, DIM, BK_INIT, false, KZ><<<grid, block, 0, s>>>(G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
        default:
            k_back<ARC, DIM, BK_UPDATE, false, KZ><<<grid, block, 0, s>>>(G, vtab, ctl, v, proj, scale, out, g, ht);
            break;
    }
}

static int back_kz() {
    static int kz = [] {
        const char* e = getenv("CTR_BK_KZ");
        const int v = e ? atoi(e) : BK_KZ_DEFAULT;
        return (v == 8 || v == 12 || v == 24 || v == 32) ? v : 16;
    }();
    return kz;
}

template <bool ARC, int DIM>
static void back_dispatch(const DGeom& G, const float4* vtab, const Ctl* ctl, Views v, const float* proj,
                          float scale, int epi, bool lz, float* out, float* g, float* ht, cudaStream_t s) {
    if (DIM != 3) return back_dispatch_kz<ARC, DIM, 1>(G, vtab, ctl, v, proj, scale, epi, lz, out, g, ht, s);
    switch (back_kz()) {
        case 8: back_dispatch_kz<ARC, DIM, 8>(G, vtab, ctl, v, proj, scale, epi, lz, out, g, ht, s); break;
        case 12: back_dispatch_kz<ARC, DIM, 12>(G, vtab, ctl, v, proj, scale, epi, lz, out, g, ht, s); break;
        case 24: back_dispatch_kz<ARC, DIM, 24>(G, vtab, ctl, v, proj, scale, epi, lz, out, g, ht, s); break;
        case 32: back_dispatch_kz<ARC, DIM, 32>(G, vtab, ctl, v, proj, scale, epi, lz, out, g, ht, s); break;
        default: back_dispatch_kz<ARC, DIM, 16>(G, vtab, ctl, v, proj, scale, epi, lz, out, g, ht, s); break;
    }
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

template <bool ARC, int DIM>
__global__ void __launch_bounds__(128) k_count(DGeom G, const float4* __restrict__ vtab, Views V,
                                               unsigned long long* __restrict__ count) {
    const int i = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * 4 + threadIdx.y;
    unsigned long long acc = 0;
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
            long long rows = 1;
            if (DIM == 3) {
                rows = 0;
                for (int k = 0; k < G.nz; k++) {
                    const float lo = fmaxf(voxel_b(f, k), 0.f), hi = fminf(voxel_b(f, k + 1), (float)G.nt);
                    if (hi > lo) rows += (long long)ceilf(hi) - (long long)floorf(lo);
                }
            }
            acc += (unsigned long long)ncz * (unsigned long long)rows;
        }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(count, acc);
}

void launch_count(const DGeom& G, const float4* vtab, Views v, unsigned long long* count, cudaStream_t s) {
    dim3 block(32, 4), grid((G.nx + 31) / 32, (G.ny + 3) / 4);
    if (G.arc) {
        if (G.dim == 3) k_count<true, 3><<<grid, block, 0, s>>>(G, vtab, v, count);
        else k_count<true, 2><<<grid, block, 0, s>>>(G, vtab, v, count);
    } else {
        if (G.dim == 3) k_count<false, 3><<<grid, block, 0, s>>>(G, vtab, v, count);
        else k_count<false, 2><<<grid, block, 0, s>>>(G, vtab, v, count);
    }
    launches_add(1);
}

}  // namespace ctr
