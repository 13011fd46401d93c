// reg_update.cu — K4 regulariser stencil (Eq. 35) and the
// fused Algorithm 1 x-update (lines 4-5), plus the small
// elementwise kernels of the solver (dist-path g/htilde update, advance of
// the Eq. 37 counter, htilde -> h, finiteness / RMS check).
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

__constant__ int c_dirs[13][3] = {
    {1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, -1, 0},
    {0, 0, 1}, {1, 0, 1}, {-1, 0, 1}, {0, 1, 1}, {0, -1, 1},
    {1, 1, 1}, {-1, 1, 1}, {1, -1, 1}, {-1, -1, 1},
};

template <int POT>
__device__ __forceinline__ void potential(float t, float inv_delta, float& dphi, float& om) {
    if (POT == 0) {          // quadratic
        dphi = t;
        om = 1.f;
    } else if (POT == 1) {   // hyperbola
        const float u = t * inv_delta;
        om = rsqrt_ftz(fmaf(u, u, 1.f));
        dphi = t * om;
    } else {                 // Fair
        om = 1.f / fmaf(fabsf(t), inv_delta, 1.f);
        dphi = t * om;
    }
}

template <int POT, int NDIRS, bool KAPPA>
__device__ __forceinline__ void stencil(const DGeom& G, const RegParams& rp, const float* __restrict__ x,
                                        const float* __restrict__ kappa, int i, int j, int k, size_t idx,
                                        float xv, float& grad, float& curv) {
    const float kj = KAPPA ? __ldg(&kappa[idx]) : 1.f;
    float gs = 0.f, cs = 0.f;
#pragma unroll
    for (int d = 0; d < NDIRS; d++) {
        const int ox = c_dirs[d][0], oy = c_dirs[d][1], oz = c_dirs[d][2];
        const long long off = (long long)oz * G.nxy + (long long)oy * G.nx + ox;
        const float b = rp.beta[d];
#pragma unroll
        for (int sgn = 0; sgn < 2; sgn++) {
            const int si = sgn ? -1 : 1;
            const int ni = i + si * ox, nj = j + si * oy, nk = k + si * oz;
            if (ni < 0 || nj < 0 || nk < 0 || ni >= G.nx || nj >= G.ny || nk >= G.nz) continue;
            const size_t nb = (size_t)((long long)idx + si * off);
            const float wgt = KAPPA ? b * kj * __ldg(&kappa[nb]) : b;
            float dphi, om;
            potential<POT>(xv - __ldg(&x[nb]), rp.inv_delta, dphi, om);
            gs = fmaf(wgt, dphi, gs);
            cs = fmaf(wgt, om, cs);
        }
    }
    grad = gs;
    curv = 2.f * cs;
}

template <int POT, int NDIRS, bool KAPPA>
__global__ void __launch_bounds__(256) k_reg(DGeom G, RegParams rp, const float* __restrict__ x,
                                             const float* __restrict__ kappa, float* __restrict__ grad,
                                             float* __restrict__ curv) {
    const int i = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * 8 + threadIdx.y;
    const int k = blockIdx.z;
    if (i >= G.nx || j >= G.ny) return;
    const size_t idx = (size_t)k * G.nxy + (size_t)j * G.nx + i;
    float gr, cv;
    stencil<POT, NDIRS, KAPPA>(G, rp, x, kappa, i, j, k, idx, __ldg(&x[idx]), gr, cv);
    grad[idx] = gr;
    if (curv) curv[idx] = cv;
}

// Potential in scaled form: tp = t / delta.  Returns omega(t) = phi'(t)/t and
// tp * omega; phi'(t) = delta * tp * omega for all three potentials.
template <int POT>
__device__ __forceinline__ float omega_scaled(float tp) {
    if (POT == 0) return 1.f;                                   // quadratic
    if (POT == 1) return rsqrt_ftz(fmaf(tp, tp, 1.f));          // hyperbola
    return __fdividef(1.f, 1.f + fabsf(tp));                    // Fair
}

// 26/8-neighbour sums over a register window W[slot][dy+1][dx+1] of x/delta
// whose planes z-1, z, z+1 sit in ring slots ZA, ZB, ZC (compile-time, so the
// z-march rotates slots instead of moving registers).  Returns
// gs = sum_n w_n tp_n omega_n and cs = sum_n w_n omega_n (w_n = beta kappa_j
// kappa_n); grad = delta gs, curv = 2 cs.  CHECK = false is the interior path:
// every neighbour exists, no predicates, and without kappa the two
// neighbours of a direction share one beta multiply.
template <int NDIRS, bool KAPPA, int POT, int ZA, int ZB, int ZC, bool CHECK>
__device__ __forceinline__ void window_stencil(const float (&W)[4][3][3], const float (&K)[4][3][3],
                                               const RegParams& rp, bool im, bool ip, bool jm, bool jp, bool km,
                                               bool kp, float& gs_out, float& cs_out) {
    const float xv = W[ZB][1][1];
    const float kj = KAPPA ? K[ZB][1][1] : 1.f;
    float gs = 0.f, cs = 0.f;
#pragma unroll
    for (int d = 0; d < NDIRS; d++) {
        const int ox = dir_x(d), oy = dir_y(d), oz = dir_z(d);
        const int zp = oz > 0 ? ZC : ZB, zm = oz > 0 ? ZA : ZB;
        if (!CHECK && !KAPPA) {
            const float tp = xv - W[zp][1 + oy][1 + ox];
            const float tm = xv - W[zm][1 - oy][1 - ox];
            const float op = omega_scaled<POT>(tp), om = omega_scaled<POT>(tm);
            gs = fmaf(rp.beta[d], fmaf(tp, op, tm * om), gs);
            cs = fmaf(rp.beta[d], op + om, cs);
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
                    const float o = omega_scaled<POT>(t);
                    gs = fmaf(wgt, t * o, gs);
                    cs = fmaf(wgt, o, cs);
                }
            }
        }
    }
    gs_out = gs;
    cs_out = cs;
}

// Fused stencil + x-update (Algorithm 1 lines 4-5).  Block = 32 consecutive i
// (a warp) x NZC z-chunks x JPB rows j; thread = one voxel column (i, j) over
// the z-chunk [c CZ, (c+1) CZ).  The 3x3 neighbourhood of x/delta (and kappa)
// of four planes lives in a register ring: plane k+2 and D_L, g, htilde of
// voxel k+1 are fetched at the top of step k and first touched one step later
// (a full stencil of latency hiding); the march is unrolled by 4 so the ring
// slots are compile-time.
// Interior columns and planes take the predicate-free stencil (warp-uniform
// except in the edge warps); the JPB rows of a block share their x rows in L1.
// x+ and htilde_partial are written in the boundary layout (coalesced over i).
// With pfx != nullptr the block also forms the z-prefix of its columns for the
// forward projector: x+ of the column tile is kept in shared memory, chunk
// totals are scanned across the NZC chunks, and each thread writes the
// entries of its chunk (float2 (P_k, x_k), z-fastest, column stride
// pfx_stride_of(G)).  32-bit element offsets (nvox < 2^32, ct_geom_create).
template <int POT, int NDIRS, bool KAPPA>
__global__ void __launch_bounds__(256) k_update(DGeom G, RegParams rp, const Ctl* __restrict__ ctl, float* xa,
                                                float* xb, const float* __restrict__ dl,
                                                const float* __restrict__ g, float* __restrict__ ht,
                                                const float* __restrict__ kappa, float box_lo, float box_hi,
                                                float* __restrict__ pfx, int CZ) {
    extern __shared__ float upd_sm[];  // pfx: xs[JPB][nz][33], tot[JPB][NZC][32]
    const int lane = threadIdx.x, c = threadIdx.y, jj = threadIdx.z;
    const int NZC = blockDim.y;
    const int i = blockIdx.x * 32 + lane;
    const int j = blockIdx.y * blockDim.z + jj;
    const bool act = i < G.nx && j < G.ny;
    const bool odd = ((ctl->k - ctl->k_base) & 1) != 0;
    const float* __restrict__ x = odd ? xb : xa;
    float* __restrict__ xn = odd ? xa : xb;
    const float rho = rho_of_k(ctl);
    const float alpha = ctl->alpha;
    const float idel = rp.inv_delta, del = rp.delta;
    const bool im = i > 0, ip = i + 1 < G.nx, jm = j > 0, jp = j + 1 < G.ny;
    const bool inxy = act && im && ip && jm && jp;
    const unsigned nx = (unsigned)G.nx, nxy = (unsigned)G.nxy;
    const unsigned col = act ? (unsigned)j * nx + (unsigned)i : 0u;
    const int k0 = c * CZ, k1 = min(G.nz, k0 + CZ);
    float* xs = upd_sm + (size_t)jj * G.nz * 33;
    float* tot = upd_sm + (size_t)blockDim.z * G.nz * 33 + (size_t)(jj * NZC) * 32;
    float W[4][3][3], K[4][3][3], XC[4];
    float Dv[2], Gv[2], Hv[2];  // D_L, g, htilde of the current / next voxel
    // raw loads into a ring slot; the slot is scaled by 1/delta one step later
    auto load_plane = [&](auto slot_c, int k) {
        constexpr int S = decltype(slot_c)::value;
        const bool ok = act && k >= 0 && k < G.nz;
        const unsigned o = ok ? (unsigned)k * nxy + col : 0u;
#pragma unroll
        for (int dy = -1; dy <= 1; dy++) {
            const bool vy = inxy || (dy < 0 ? jm : (dy > 0 ? jp : true));
            const unsigned ro = o + (unsigned)(dy * (int)nx);
#pragma unroll
            for (int dx = -1; dx <= 1; dx++) {
                const bool v = ok && vy && (inxy || (dx < 0 ? im : (dx > 0 ? ip : true)));
                W[S][dy + 1][dx + 1] = v ? __ldg(x + (ro + (unsigned)dx)) : 0.f;
                if (KAPPA) K[S][dy + 1][dx + 1] = v ? __ldg(kappa + (ro + (unsigned)dx)) : 0.f;
            }
        }
    };
    auto scale_plane = [&](auto slot_c) {
        constexpr int S = decltype(slot_c)::value;
        XC[S] = W[S][1][1];
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int b = 0; b < 3; b++) W[S][a][b] *= idel;
    };
    auto load_vox = [&](auto par_c, int k) {
        constexpr int Q = decltype(par_c)::value;
        const bool ok = act && k < k1;
        const unsigned idx = ok ? (unsigned)k * nxy + col : 0u;
        Dv[Q] = ok ? __ldg(dl + idx) : 0.f;
        Gv[Q] = ok ? __ldg(g + idx) : 0.f;
        Hv[Q] = ok ? ht[idx] : 0.f;
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
        load_vox(std::integral_constant<int, Q ^ 1>(), k + 1);
        float xnew = 0.f;
        if (act) {
            const unsigned idx = (unsigned)k * nxy + col;
            float gs, cs;
            const bool km = k > 0, kp = k + 1 < G.nz;
            if (inxy && km && kp)
                window_stencil<NDIRS, KAPPA, POT, ZA, ZB, ZC, false>(W, K, rp, im, ip, jm, jp, km, kp, gs, cs);
            else
                window_stencil<NDIRS, KAPPA, POT, ZA, ZB, ZC, true>(W, K, rp, im, ip, jm, jp, km, kp, gs, cs);
            const float xv = XC[ZB];
            const float d = Dv[Q], htv = Hv[Q];
            const float s = fmaf(rho, htv, (1.f - rho) * Gv[Q]);
            const float den = fmaf(rho, d, 2.f * cs);
            xnew = xv;
            if (den > 0.f) xnew = fminf(fmaxf(xv - __fdividef(fmaf(del, gs, s), den), box_lo), box_hi);
            xn[idx] = xnew;
            ht[idx] = (1.f - alpha) * fmaf(d, xnew - xv, htv);
        }
        if (pfx) {
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
    load_vox(I1(), k0);
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
    if (!pfx) return;
    tot[c * 32 + lane] = run;
    __syncthreads();
    float P = 0.f;
    for (int q = 0; q < c; q++) P += tot[q * 32 + lane];
    if (!act) return;
    float2* __restrict__ pc = reinterpret_cast<float2*>(pfx) + (size_t)col * (size_t)pfx_stride_of(G);
    for (int k = k0; k < k1; k++) {
        const float xk = xs[k * 33 + lane];
        pc[k] = make_float2(P, xk);  // (P_k, x_k): prefix before voxel k and the voxel
        P += xk;
    }
    if (k1 == G.nz) pc[G.nz] = make_float2(P, 0.f);  // (P_nz, 0)
}

template <int POT, int NDIRS>
static void reg_dispatch(const DGeom& G, const RegParams& rp, const float* x, const float* kappa, float* grad,
                         float* curv, cudaStream_t s) {
    dim3 block(32, 8), grid((G.nx + 31) / 32, (G.ny + 7) / 8, G.nz);
    if (kappa) k_reg<POT, NDIRS, true><<<grid, block, 0, s>>>(G, rp, x, kappa, grad, curv);
    else k_reg<POT, NDIRS, false><<<grid, block, 0, s>>>(G, rp, x, kappa, grad, curv);
}

void launch_reg(const DGeom& G, const RegParams& rp, const float* x, const float* kappa, float* grad, float* curv,
                cudaStream_t s) {
    const bool d4 = rp.n_dirs == 4;
    switch (rp.potential) {
        case 0: d4 ? reg_dispatch<0, 4>(G, rp, x, kappa, grad, curv, s) : reg_dispatch<0, 13>(G, rp, x, kappa, grad, curv, s); break;
        case 1: d4 ? reg_dispatch<1, 4>(G, rp, x, kappa, grad, curv, s) : reg_dispatch<1, 13>(G, rp, x, kappa, grad, curv, s); break;
        default: d4 ? reg_dispatch<2, 4>(G, rp, x, kappa, grad, curv, s) : reg_dispatch<2, 13>(G, rp, x, kappa, grad, curv, s); break;
    }
    launches_add(1);
}

// launch shape of k_update: NZC z-chunks of CZ voxels, JPB rows per block (<= 256 threads)
struct UpdShape {
    int nzc, cz, jpb;
    size_t smem;
};
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

static UpdShape upd_shape(const DGeom& G, bool pfx) {
    UpdShape u;
    static const int zdiv = env_int("CTR_UPD_ZDIV", 32);  // tuning knob: voxels per z-chunk target
    u.nzc = std::min(8, std::max(1, G.nz / std::max(1, zdiv)));
    u.cz = (G.nz + u.nzc - 1) / u.nzc;
    u.nzc = (G.nz + u.cz - 1) / u.cz;
    u.jpb = std::max(1, 8 / u.nzc);  // JPB rows per block share x rows in L1
    u.smem = pfx ? sizeof(float) * ((size_t)u.jpb * G.nz * 33 + (size_t)u.jpb * u.nzc * 32) : 0;
    return u;
}

size_t update_smem_bytes(const DGeom& G) { return upd_shape(G, true).smem; }

template <int POT, int NDIRS>
static void upd_dispatch(const DGeom& G, const RegParams& rp, const Ctl* ctl, float* xa, float* xb, const float* dl,
                         const float* g, float* ht, const float* kappa, float lo, float hi, float* pfx,
                         cudaStream_t s) {
    static const int nopfx = env_int("CTR_UPD_NOPFX", 0);  // timing experiment only: skips the prefix
    if (nopfx) pfx = nullptr;
    const UpdShape u = upd_shape(G, pfx != nullptr);
    dim3 block(32, u.nzc, u.jpb), grid((G.nx + 31) / 32, (G.ny + u.jpb - 1) / u.jpb, 1);
    if (kappa) {
        if (u.smem > 48 * 1024)
            cudaFuncSetAttribute(k_update<POT, NDIRS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)u.smem);
        k_update<POT, NDIRS, true><<<grid, block, u.smem, s>>>(G, rp, ctl, xa, xb, dl, g, ht, kappa, lo, hi, pfx, u.cz);
    } else {
        if (u.smem > 48 * 1024)
            cudaFuncSetAttribute(k_update<POT, NDIRS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)u.smem);
        k_update<POT, NDIRS, false><<<grid, block, u.smem, s>>>(G, rp, ctl, xa, xb, dl, g, ht, kappa, lo, hi, pfx, u.cz);
    }
}

void launch_update(const DGeom& G, const RegParams& rp, const Ctl* ctl, float* xa, float* xb, const float* dl,
                   const float* g, float* ht, const float* kappa, float box_lo, float box_hi, float* pfx,
                   cudaStream_t s) {
    const bool d4 = rp.n_dirs == 4;
    switch (rp.potential) {
        case 0: d4 ? upd_dispatch<0, 4>(G, rp, ctl, xa, xb, dl, g, ht, kappa, box_lo, box_hi, pfx, s) : upd_dispatch<0, 13>(G, rp, ctl, xa, xb, dl, g, ht, kappa, box_lo, box_hi, pfx, s); break;
        case 1: d4 ? upd_dispatch<1, 4>(G, rp, ctl, xa, xb, dl, g, ht, kappa, box_lo, box_hi, pfx, s) : upd_dispatch<1, 13>(G, rp, ctl, xa, xb, dl, g, ht, kappa, box_lo, box_hi, pfx, s); break;
        default: d4 ? upd_dispatch<2, 4>(G, rp, ctl, xa, xb, dl, g, ht, kappa, box_lo, box_hi, pfx, s) : upd_dispatch<2, 13>(G, rp, ctl, xa, xb, dl, g, ht, kappa, box_lo, box_hi, pfx, s); break;
    }
    launches_add(1);
}

// ---- small elementwise kernels ----
__global__ void k_gh_update(long long n, const Ctl* __restrict__ ctl, const float* __restrict__ zeta, float* g,
                            float* ht) {
    const float rho = rho_of_k(ctl), alpha = ctl->alpha, inv = 1.f / (rho + 1.f);
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        const float z = zeta[idx], gv = g[idx];
        g[idx] = fmaf(rho * inv, fmaf(alpha, z, (1.f - alpha) * gv), gv * inv);
        ht[idx] = fmaf(alpha, z, ht[idx]);
    }
}

__global__ void k_init_from_zeta(long long n, const float* __restrict__ zeta, float* g, float* ht) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        g[idx] = zeta[idx];
        ht[idx] = zeta[idx];
    }
}

__global__ void k_advance(Ctl* ctl) { ctl->k += 1; }

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
void launch_advance(Ctl* ctl, cudaStream_t s) {
    k_advance<<<1, 1, 0, s>>>(ctl);
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
