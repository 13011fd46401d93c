// fbp.cu — FBP / FDK initialiser (PAPER.md:334 starts
// Algorithm 1 from "an initial (FBP) image").  Textbook fan-beam FBP
// (equiangular arc / equispaced flat) and its Feldkamp extension for axial
// cone scans, the same steps as oracle/fbp.py:
//   k_fbp_filter: pre-weight (flat D/sqrt(D^2+s^2+t^2), arc D cos(gamma)
//     D/sqrt(D^2+t^2)) and Ram-Lak filtering of every detector row, one block
//     per (view, row), the weighted row staged in shared memory.
//   k_fbp_back: voxel-driven back-projection, thread = voxel column (the
//     transaxial position, weight and column coordinate of a view are shared
//     by the column's voxels), bilinear interpolation, (2 pi / na) sum.
#include "kernels.cuh"

namespace ctr {

constexpr int FB_BS = 256;

template <bool ARC>
__global__ void __launch_bounds__(FB_BS) k_fbp_filter(DGeom G, const float* __restrict__ proj, float* __restrict__ q,
                                                      float dv, float vscale) {
    extern __shared__ float fsm[];  // weighted row (ns), then the taps h[m], m = -(ns-1)..ns-1
    const int t = blockIdx.x, v = blockIdx.y;
    const int ns = G.ns;
    float* rw = fsm;
    float* hk = fsm + ns + (ns - 1);   // hk[m] for |m| < ns
    const float D = G.dso;
    const float th = ((float)t + 0.5f - G.t_c0p) * G.dt;   // row centre at the detector
    const float tv = th * vscale;                           // on the virtual detector through the isocentre
    const float* __restrict__ row = proj + ((size_t)v * G.nt + t) * ns;
    for (int s = threadIdx.x; s < ns; s += FB_BS) {
        const float sig = ((float)s - G.s_c0) * G.delta;
        float w;
        if (ARC) {
            w = D * cosf(sig) * D * rsqrtf(fmaf(tv, tv, D * D));
        } else {
            const float sv = sig * vscale;
            w = D * rsqrtf(fmaf(sv, sv, fmaf(tv, tv, D * D)));
        }
        rw[s] = __ldg(&row[s]) * w;
    }
    // Ram-Lak taps: h[0] = 1/(4 dv^2); odd m: -1/(pi^2 m^2 dv^2) (flat), -1/(pi^2 sin^2(m dv)) (arc); even 0
    const float c = 1.f / (3.14159265358979f * 3.14159265358979f);
    for (int m = threadIdx.x; m < ns; m += FB_BS) {
        float hm = 0.f;
        if (m == 0) {
            hm = 0.25f / (dv * dv);
        } else if (m & 1) {
            if (ARC) {
                const float sn = sinf((float)m * dv);
                hm = -c / (sn * sn);
            } else {
                hm = -c / ((float)m * (float)m * dv * dv);
            }
        }
        hk[m] = hm;
        hk[-m] = hm;
    }
    __syncthreads();
    float* __restrict__ out = q + ((size_t)v * G.nt + t) * ns;
    for (int n = threadIdx.x; n < ns; n += FB_BS) {
        float acc = rw[n] * hk[0];
        for (int k = (n & 1) ? 0 : 1; k < ns; k += 2) acc = fmaf(rw[k], hk[n - k], acc);   // odd n - k only
        out[n] = 0.5f * dv * acc;
    }
}

template <bool ARC, int DIM>
__global__ void __launch_bounds__(FB_BS) k_fbp_back(DGeom G, const float4* __restrict__ vtab,
                                                    const float* __restrict__ q, float scale, float vscale,
                                                    float* __restrict__ out) {
    const int i = blockIdx.x * 32 + (threadIdx.x & 31);
    const int j = blockIdx.y * (FB_BS / 32) + (threadIdx.x >> 5);
    if (i >= G.nx || j >= G.ny) return;
    const float D = G.dso;
    const float cx = fmaf((float)i, G.dx, G.x0), cy = fmaf((float)j, G.dy, G.y0);
    const int nz = DIM == 3 ? G.nz : 1, nt = DIM == 3 ? G.nt : 1;
    const float rowpitch = G.dt * vscale;   // virtual-detector row pitch
    const float tc0 = G.t_c0p - 0.5f;       // fractional row of t = 0
    constexpr int KMAX = 16;                 // z voxels per register block
    for (int kb = 0; kb < nz; kb += KMAX) {
        float acc[KMAX];
#pragma unroll
        for (int q2 = 0; q2 < KMAX; q2++) acc[q2] = 0.f;
        for (int v = 0; v < G.na; v++) {
            const float4 vw = __ldg(&vtab[v]);
            const float cb = vw.x, sb = vw.y, zs = vw.z;
            const float rx = fmaf(-D, cb, cx), ry = fmaf(-D, sb, cy);
            const float a = -(rx * cb + ry * sb);
            const float b = ry * cb - rx * sb;
            float ucol, wgt, tsc;
            if (ARC) {
                const float L2 = fmaf(rx, rx, ry * ry);
                ucol = atan2f(b, a) * G.inv_delta + G.s_c0;
                wgt = 1.f / L2;
                tsc = D * rsqrtf(L2) / rowpitch;       // t' = D (z - z_s)/L in rows
            } else {
                const float ia = 1.f / a;
                ucol = D * b * ia / (G.delta * vscale) + G.s_c0;
                wgt = D * D * ia * ia;
                tsc = D * ia / rowpitch;
            }
            const float fc = floorf(ucol);
            const int c0 = (int)fc;
            const float wc = ucol - fc;
            if (c0 < -1 || c0 >= G.ns) continue;
            const float* __restrict__ qv = q + (size_t)v * nt * G.ns;
            const bool okl = c0 >= 0, okr = c0 + 1 < G.ns;
#pragma unroll
            for (int q2 = 0; q2 < KMAX; q2++) {
                const int k = kb + q2;
                if (k >= nz) break;
                float val;
                if (DIM == 3) {
                    const float z = fmaf((float)k, G.dz, G.z0);
                    const float ur = fmaf(z - zs, tsc, tc0);
                    const float fr = floorf(ur);
                    const int r0 = (int)fr;
                    const float wr = ur - fr;
                    float v00 = 0.f, v01 = 0.f, v10 = 0.f, v11 = 0.f;
                    if (r0 >= 0 && r0 < nt) {
                        const float* pr = qv + (size_t)r0 * G.ns;
                        if (okl) v00 = __ldg(&pr[c0]);
                        if (okr) v01 = __ldg(&pr[c0 + 1]);
                    }
                    if (r0 + 1 >= 0 && r0 + 1 < nt) {
                        const float* pr = qv + (size_t)(r0 + 1) * G.ns;
                        if (okl) v10 = __ldg(&pr[c0]);
                        if (okr) v11 = __ldg(&pr[c0 + 1]);
                    }
                    val = (1.f - wr) * fmaf(wc, v01 - v00, v00) + wr * fmaf(wc, v11 - v10, v10);
                } else {
                    const float v0 = okl ? __ldg(&qv[c0]) : 0.f, v1 = okr ? __ldg(&qv[c0 + 1]) : 0.f;
                    val = fmaf(wc, v1 - v0, v0);
                }
                acc[q2] = fmaf(wgt, val, acc[q2]);
            }
        }
#pragma unroll
        for (int q2 = 0; q2 < KMAX; q2++) {
            const int k = kb + q2;
            if (k < nz) out[(size_t)k * G.nxy + (size_t)j * G.nx + i] = scale * acc[q2];
        }
    }
}

void launch_fbp(const DGeom& G, const float4* vtab, const float* proj, float* qbuf, float* out, double dsd,
                cudaStream_t s) {
    const float vscale = (float)(G.dso / dsd);             // detector -> virtual detector at the isocentre
    const float dv = G.arc ? G.delta : G.delta * vscale;    // filter sampling interval
    dim3 gf(G.nt, G.na);
    const size_t smem = sizeof(float) * (3 * (size_t)G.ns - 1);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(k_fbp_filter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fbp_filter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (G.arc) k_fbp_filter<true><<<gf, FB_BS, smem, s>>>(G, proj, qbuf, dv, vscale);
    else k_fbp_filter<false><<<gf, FB_BS, smem, s>>>(G, proj, qbuf, dv, vscale);
    dim3 gb((G.nx + 31) / 32, (G.ny + FB_BS / 32 - 1) / (FB_BS / 32));
    const float scale = (float)(2.0 * 3.14159265358979323846 / G.na);
    if (G.arc) {
        if (G.dim == 3) k_fbp_back<true, 3><<<gb, FB_BS, 0, s>>>(G, vtab, qbuf, scale, vscale, out);
        else k_fbp_back<true, 2><<<gb, FB_BS, 0, s>>>(G, vtab, qbuf, scale, vscale, out);
    } else {
        if (G.dim == 3) k_fbp_back<false, 3><<<gb, FB_BS, 0, s>>>(G, vtab, qbuf, scale, vscale, out);
        else k_fbp_back<false, 2><<<gb, FB_BS, 0, s>>>(G, vtab, qbuf, scale, vscale, out);
    }
    launches_add(2);
}

}  // namespace ctr
