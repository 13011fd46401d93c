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
        om = rsqrtf(fmaf(u, u, 1.f));
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

template <int NDIRS, bool KAPPA, int POT>
__device__ __forceinline__ void window_stencil(const float (&W)[3][3][3], const float (&K)[3][3][3],
                                               const RegParams& rp, bool im, bool ip, bool jm, bool jp, bool km,
                                               bool kp, float& grad, float& curv) {
    const float xv = W[1][1][1];
    const float kj = KAPPA ? K[1][1][1] : 1.f;
    float gs = 0.f, cs = 0.f;
#pragma unroll
    for (int d = 0; d < NDIRS; d++) {
#pragma unroll
        for (int sg = 0; sg < 2; sg++) {
            const int ox = sg ? -dir_x(d) : dir_x(d);
            const int oy = sg ? -dir_y(d) : dir_y(d);
            const int oz = sg ? -dir_z(d) : dir_z(d);
            const bool ok = (ox < 0 ? im : (ox > 0 ? ip : true)) && (oy < 0 ? jm : (oy > 0 ? jp : true)) &&
                            (oz < 0 ? km : (oz > 0 ? kp : true));
            if (ok) {
                const float wgt = KAPPA ? rp.beta[d] * kj * K[1 + oz][1 + oy][1 + ox] : rp.beta[d];
                float dphi, om;
                potential<POT>(xv - W[1 + oz][1 + oy][1 + ox], rp.inv_delta, dphi, om);
                gs = fmaf(wgt, dphi, gs);
                cs = fmaf(wgt, om, cs);
            }
        }
    }
    grad = gs;
    curv = 2.f * cs;
}

// Fused stencil + x-update, z-marching: thread = one voxel column (i, j), all
// nz voxels; a warp = 32 consecutive i at one j.  The 3x3x3 neighbourhood of x
// (and kappa) lives in registers and advances one plane per voxel (9 loads per
// voxel instead of 27).  x+ and htilde_partial are written in the boundary
// layout (coalesced over i).  With pfx != nullptr the thread also forms the
// z-prefix P_k = sum_{k'<k} x+_k' of its column for the forward projector;
// 32 prefix values per column are staged in shared memory and written as
// whole 128-byte lines (z-fastest layout, column stride pfx_stride_of(G)).
template <int POT, int NDIRS, bool KAPPA>
__global__ void __launch_bounds__(128) k_update(DGeom G, RegParams rp, const Ctl* __restrict__ ctl, float* xa,
                                                float* xb, const float* __restrict__ dl,
                                                const float* __restrict__ g, float* __restrict__ ht,
                                                const float* __restrict__ kappa, float box_lo, float box_hi,
                                                float* __restrict__ pfx) {
    __shared__ float pst[4][32][33];
    const int lane = threadIdx.x, wy = threadIdx.y;
    const int i = blockIdx.x * 32 + lane;
    const int j = blockIdx.y * 4 + wy;
    const bool act = i < G.nx && j < G.ny;
    if (j >= G.ny) return;  // warp-uniform (whole warp shares j)
    const bool odd = ((ctl->k - ctl->k_base) & 1) != 0;
    const float* __restrict__ x = odd ? xb : xa;
    float* __restrict__ xn = odd ? xa : xb;
    const float rho = rho_of_k(ctl);
    const float alpha = ctl->alpha;
    const bool im = i > 0, ip = i + 1 < G.nx, jm = j > 0, jp = j + 1 < G.ny;
    const size_t col = (size_t)j * G.nx + (act ? i : 0);
    const int ps = pfx_stride_of(G);
    float W[3][3][3], K[3][3][3];
    auto load_plane = [&](int slot, int k) {
        const bool ok = act && k >= 0 && k < G.nz;
#pragma unroll
        for (int dy = -1; dy <= 1; dy++) {
#pragma unroll
            for (int dx = -1; dx <= 1; dx++) {
                const bool v = ok && (dx < 0 ? im : (dx > 0 ? ip : true)) && (dy < 0 ? jm : (dy > 0 ? jp : true));
                const size_t a = (size_t)k * G.nxy + col + (long long)dy * G.nx + dx;
                W[slot][dy + 1][dx + 1] = v ? __ldg(&x[a]) : 0.f;
                if (KAPPA) K[slot][dy + 1][dx + 1] = v ? __ldg(&kappa[a]) : 0.f;
            }
        }
    };
    auto flush = [&](int kb, int n) {  // prefix entries kb .. kb+n-1 of the warp's 32 columns
        __syncwarp();
        const int cbase = blockIdx.x * 32;
        for (int c = 0; c < 32; c++) {
            if (cbase + c < G.nx && lane < n)
                pfx[((size_t)j * G.nx + cbase + c) * ps + kb + lane] = pst[wy][lane][c];
        }
        __syncwarp();
    };
    load_plane(1, -1);
    load_plane(2, 0);
    float run = 0.f;
    int kb = 0, cnt = 0;
    auto push = [&](float v) {
        pst[wy][cnt][lane] = v;
        if (++cnt == 32) {
            flush(kb, 32);
            kb += 32;
            cnt = 0;
        }
    };
    for (int k = 0; k < G.nz; k++) {
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int b = 0; b < 3; b++) {
                W[0][a][b] = W[1][a][b];
                W[1][a][b] = W[2][a][b];
                if (KAPPA) {
                    K[0][a][b] = K[1][a][b];
                    K[1][a][b] = K[2][a][b];
                }
            }
        load_plane(2, k + 1);
        float xnew = 0.f;
        if (act) {
            float gr, cv;
            window_stencil<NDIRS, KAPPA, POT>(W, K, rp, im, ip, jm, jp, k > 0, k + 1 < G.nz, gr, cv);
            const size_t idx = (size_t)k * G.nxy + col;
            const float xv = W[1][1][1];
            const float d = __ldg(&dl[idx]);
            const float htv = ht[idx];
            const float s = fmaf(rho, htv, (1.f - rho) * __ldg(&g[idx]));
            const float den = fmaf(rho, d, cv);
            xnew = xv;
            if (den > 0.f) xnew = fminf(fmaxf(xv - (s + gr) / den, box_lo), box_hi);
            xn[idx] = xnew;
            ht[idx] = (1.f - alpha) * fmaf(d, xnew - xv, htv);
        }
        if (pfx) {
            push(run);   // P_k: prefix before voxel k
            run += xnew;
        }
    }
    if (pfx) {
        push(run);  // P_nz
        push(run);  // P_nz+1 = P_nz (padding read by the forward's interpolation)
        if (cnt) flush(kb, cnt);
    }
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

template <int POT, int NDIRS>
static void upd_dispatch(const DGeom& G, const RegParams& rp, const Ctl* ctl, float* xa, float* xb, const float* dl,
                         const float* g, float* ht, const float* kappa, float lo, float hi, float* pfx,
                         cudaStream_t s) {
    dim3 block(32, 4), grid((G.nx + 31) / 32, (G.ny + 3) / 4, 1);
    if (kappa) k_update<POT, NDIRS, true><<<grid, block, 0, s>>>(G, rp, ctl, xa, xb, dl, g, ht, kappa, lo, hi, pfx);
    else k_update<POT, NDIRS, false><<<grid, block, 0, s>>>(G, rp, ctl, xa, xb, dl, g, ht, kappa, lo, hi, pfx);
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
