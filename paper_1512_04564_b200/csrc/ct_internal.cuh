// ct_internal.cuh — device-side geometry and separable-footprint (SF) helpers
// shared by the forward and back-projection kernels of libctrecon.so.
//
// The projector is the SF model of DESIGN.md §3; the paper
// only cites it (PAPER.md:315 [long:10:3fa]).  Forward and back projection
// call the SAME footprint function (ct_footprint) and the same trapezoid
// antiderivative (trap_T), so the GPU A' is the transpose of the GPU A up to
// summation order.
//
// float32 numerics: corner footprints are computed relative to the column
// centre (cross/dot of the centre ray with the corner offset), so the
// trapezoid breakpoints are formed from O(voxel) numbers instead of
// differences of large absolute angles / detector positions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Device-side bounds checks for a debug build (-DCTR_DEBUG_CHECKS; compute-sanitizer is not
// available on the GPU pool): every gather offset and shared-memory index the kernels compute
// is checked against its array's extent, and a failure traps (the launch fails loudly).
#ifdef CTR_DEBUG_CHECKS
#include <cstdio>
#define CTR_CHECK(cond, what)                                                                            \
    do {                                                                                                 \
        if (!(cond)) {                                                                                   \
            printf("CTR_CHECK failed: %s (%s:%d) block (%d,%d,%d) thread (%d,%d,%d)\n", what, __FILE__,   \
                   __LINE__, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, threadIdx.y, threadIdx.z);  \
            __trap();                                                                                    \
        }                                                                                                \
    } while (0)
#else
#define CTR_CHECK(cond, what) \
    do {                      \
    } while (0)
#endif

namespace ctr {

constexpr int kMaxCells = 16;     // max detector columns under one voxel footprint
constexpr float kRampEps = 1e-6f; // ramp widths below this (in cells) take their limit

struct DGeom {
    int dim, nx, ny, nz, ns, nt, arc, na;
    float dx, dy, dz;
    float x0, y0, z0;     // centre of voxel (0,0,0)
    float delta;          // column pitch: mm (flat) or rad (arc)
    float inv_delta;
    float s_c0;           // (ns-1)/2 + offset_s: fractional column of tau = 0
    float t_c0p;          // (nt-1)/2 + offset_t + 1/2: row units, row t spans [t, t+1)
    float dt, inv_dt, dso, dsd;
    float zbot, ztop;     // z-extent of the volume (voxel edges)
    float rxy;            // radius of the volume's circumscribed cylinder (incl. offsets)
    float zs0, zstep;     // source z of view v: zs0 + v zstep (helical; zstep = 0 axial)
    long long nxy, nvox;
};

// Solver control block in device memory (read by every kernel of a captured
// sub-iteration; advanced by k_advance).  Views of the current subset and
// rho are derived on the device from k, so one CUDA graph serves every
// sub-iteration.
struct Ctl {
    long long k;        // sub-iterations done (Eq. 37 counter)
    long long k_base;   // k at the start of this solve call (x buffer parity)
    int M, na;
    int rank, world;    // view sharding (dist), 0/1 on a single GPU
    int rho_fixed_mode;
    int simple;         // Algorithm 2: the htilde array holds zeta
    float alpha, rho_fixed;
    int bad;            // set by kernels on footprint overflow (debug guard)
    unsigned done;      // blocks of the current back-projection finished (advance_after_last_block)
};

// Algorithm 1 line 9 (k <- k + 1) folded into the back-projection that ends a
// sub-iteration: the last block to finish advances the counter and resets the block count
// (no separate one-thread launch).  Every thread of every block must reach this call; the
// other blocks' reads of k (view selection, rho) are complete by then.
__device__ __forceinline__ void advance_after_last_block(const Ctl* ctl) {
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0) {
        Ctl* c = const_cast<Ctl*>(ctl);
        __threadfence();
        const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
        if (atomicAdd(&c->done, 1u) == nb - 1) {
            c->done = 0;
            c->k += 1;
            __threadfence();
        }
    }
}

struct Views {          // explicit descriptor, or subset-from-Ctl when ctl != nullptr
    int start, stride, count;
};

__device__ __forceinline__ float rho_at(const Ctl* c, long long k) {
    if (c->rho_fixed_mode) return c->rho_fixed;
    if (k == 0) return 1.0f;
    double a = 3.14159265358979323846 / ((double)c->alpha * (double)(k + 1));
    double b = 0.5 * a;
    return (float)(a * sqrt(1.0 - b * b));
}

__device__ __forceinline__ float rho_of_k(const Ctl* c) { return rho_at(c, c->k); }

// View selection: subset m = k mod M, sharded over ranks (rank p takes the
// subset-local views p, p+G, ...).
__device__ __forceinline__ Views select_views(const Ctl* c, Views v) {
    if (!c) return v;
    int m = (int)(c->k % c->M);
    int vm = (c->na - m + c->M - 1) / c->M;
    Views o;
    o.start = m + c->rank * c->M;
    o.stride = c->world * c->M;
    o.count = (vm - c->rank + c->world - 1) / c->world;
    if (o.count < 0) o.count = 0;
    return o;
}

// MUFU.RSQ without the denormal fix-up rsqrtf() carries (3 extra instructions):
// every call site passes an argument >= 1 (potential weights) or a squared
// distance of millimetres (footprints), never a denormal.
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// 1/x in one MUFU.RCP (no denormal-divisor fix-up: callers pass x > 0 well above 2^-126)
__device__ __forceinline__ float rcp_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// L2 evict-last policy for data re-read by many views (the forward's z-prefix
// array) and a gather that carries it; streaming (evict-first) for data read
// or written once per sub-iteration goes through __ldcs / __stcs.
__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float ldg_keep(const float* p, unsigned long long pol) {
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// Packed FP32 (sm_100a FFMA2 / FADD2 / FMUL2: two IEEE float32 operations per lane in one
// instruction, the same rounding as the scalar ones).  A scalar operand duplicated into both
// halves folds into the instruction's broadcast form (no extra move).
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 bcast2(float a) { return make_float2(a, a); }

__device__ __forceinline__ void sort4(float& a, float& b, float& c, float& d) {
    float t;
#define CTR_CS(p, q) if (p > q) { t = p; p = q; q = t; }
    CTR_CS(a, b) CTR_CS(c, d) CTR_CS(a, c) CTR_CS(b, d) CTR_CS(b, c)
#undef CTR_CS
}

// Per (view, voxel column) footprint.
struct Footprint {
    float sfc;            // fractional column index of the column centre's tau
    float u0, u1, u2, u3; // sorted corner taus relative to the centre, in columns
    float inv2r1, halfr2, inv2r2;  // trapezoid ramp constants (0 if degenerate)
    float lxy;            // transaxial amplitude L_xy
    float B0, H;          // axial: voxel k spans row units [B0 + k H, B0 + (k+1) H]
};

// view: (cos beta, sin beta, z_s)
// Arithmetic: the column centre's tau uses IEEE division and atan_pos (it sets
// the absolute position of the footprint on the detector); the corner offsets are
// O(voxel) quantities, computed as atan(z) ~ z - z^3/3 + z^5/5 of z = cross/dot
// (|z| < 0.05 in every supported geometry: truncation < 1e-8 relative) and
// with fast reciprocals (__fdividef, rsqrtf: 2 ulp) -- DESIGN.md §5.
//
// The footprint is evaluated in three parts so that the back-projector can
// test the cheap axial extent before paying for the transaxial corners:
// fp_base (source-to-column vector in the view frame), fp_axial (B0, H) and
// fp_trans (corner taus, ramps, L_xy).  ct_footprint = all three; every caller
// (forward, back, nnz count) runs the same expressions.
// atan(b / a) for a > 0 (the source-to-voxel vector always points into the
// fan: a >= dso - rmax > 0, ct_geom_create).  Cephes-style reduction of
// |b|/a to |x| <= tan(pi/8) and a degree-9 odd polynomial (about 1e-7
// relative), branch-free; IEEE division keeps the column-centre position as
// accurate as atan2f at a third of its instructions.
__device__ __forceinline__ float atan_pos(float b, float a) {
    const float ab = fabsf(b);
    const bool big = ab > 2.414213562373095f * a, mid = ab > 0.4142135623730950f * a;
    const float num = big ? -a : (mid ? ab - a : ab);
    const float den = big ? ab : (mid ? ab + a : a);
    const float x = num / den;
    const float y0 = big ? 1.5707963267948966f : (mid ? 0.7853981633974483f : 0.f);
    const float z = x * x;
    const float p = fmaf(fmaf(fmaf(fmaf(8.05374449538e-2f, z, -1.38776856032e-1f), z, 1.99777106478e-1f), z,
                              -3.33329491539e-1f), z * x, x);
    return copysignf(y0 + p, b);
}

struct FpBase {
    float rx, ry;     // column centre - source (world xy)
    float a, b;       // the same in the view frame (e_c, e_u)
    float r2, rinv;   // |r|^2, 1/|r|
    float inva;       // 1/a
};

__device__ __forceinline__ void fp_base(const DGeom& G, float cb, float sb, int i, int j, FpBase& q) {
    const float cx = fmaf((float)i, G.dx, G.x0);
    const float cy = fmaf((float)j, G.dy, G.y0);
    q.rx = fmaf(-G.dso, cb, cx);
    q.ry = fmaf(-G.dso, sb, cy);
    // frame of the view: a along e_c = -(cos,sin), b along e_u = (-sin, cos)
    q.a = -(q.rx * cb + q.ry * sb);
    q.b = q.ry * cb - q.rx * sb;
    q.r2 = fmaf(q.a, q.a, q.b * q.b);
    q.rinv = rsqrt_ftz(q.r2);
    q.inva = __fdividef(1.f, q.a);
}

// axial magnification: flat Dsd/a, arc Dsd/|r|; row units u = t/dt + t_c0p;
// voxel k spans row units [B0 + k H, B0 + (k+1) H]
template <bool ARC>
__device__ __forceinline__ void fp_axial(const DGeom& G, const FpBase& q, float zs, float& B0, float& H) {
    const float mag = ARC ? G.dsd * q.rinv : G.dsd * q.inva;
    const float mdt = mag * G.inv_dt;
    H = G.dz * mdt;
    B0 = fmaf(G.z0 - 0.5f * G.dz - zs, mdt, G.t_c0p);
}

template <bool ARC>
__device__ __forceinline__ void fp_trans(const DGeom& G, float cb, float sb, const FpBase& q, Footprint& f) {
    const float a = q.a, b = q.b;
    const float hx = 0.5f * G.dx, hy = 0.5f * G.dy;
    // corner offsets (+-hx, +-hy) in (a, b): da = -(ex cb + ey sb), db = ey cb - ex sb
    const float da1 = hx * cb, da2 = hy * sb;
    const float db1 = hx * sb, db2 = hy * cb;
    float t[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const float sx = (c & 1) ? 1.f : -1.f;
        const float sy = (c & 2) ? 1.f : -1.f;
        const float dA = -(sx * da1 + sy * da2);
        const float dB = sy * db2 - sx * db1;
        const float cr = a * dB - b * dA;
        if (ARC) {
            // angle(p_k) - angle(p_c) = atan(cr / (a (a + da) + b (b + db)))
            const float z = __fdividef(cr, q.r2 + fmaf(a, dA, b * dB));
            const float z2 = z * z;
            t[c] = z * fmaf(z2, fmaf(z2, 0.2f, -0.33333334f), 1.f);
        } else {
            // Dsd (b+db)/(a+da) - Dsd b/a = Dsd (db a - b da) / (a (a + da))
            t[c] = G.dsd * cr * q.inva * __fdividef(1.f, a + dA);
        }
    }
    const float tc = ARC ? atan_pos(b, a) : G.dsd * b / a;
    sort4(t[0], t[1], t[2], t[3]);
    f.u0 = t[0] * G.inv_delta;
    f.u1 = t[1] * G.inv_delta;
    f.u2 = t[2] * G.inv_delta;
    f.u3 = t[3] * G.inv_delta;
    f.sfc = fmaf(tc, G.inv_delta, G.s_c0);
    const float w1 = f.u1 - f.u0, w2 = f.u3 - f.u2;
    f.inv2r1 = w1 > kRampEps ? __fdividef(0.5f, w1) : 0.f;
    f.halfr2 = w2 > kRampEps ? 0.5f * w2 : 0.f;
    f.inv2r2 = w2 > kRampEps ? __fdividef(0.5f, w2) : 0.f;
    // L_xy = min(dx/|d_x|, dy/|d_y|) with d = (rx, ry)/|r|, |r| = |(a, b)|
    const float rn = q.r2 * q.rinv;
    const float arx = fabsf(q.rx), ary = fabsf(q.ry);
    const float lx = arx > 0.f ? __fdividef(G.dx * rn, arx) : 3.0e38f;
    const float ly = ary > 0.f ? __fdividef(G.dy * rn, ary) : 3.0e38f;
    f.lxy = fminf(lx, ly);
}

template <bool ARC>
__device__ __forceinline__ void ct_footprint(const DGeom& G, float cb, float sb, float zs, int i, int j,
                                             Footprint& f) {
    FpBase q;
    fp_base(G, cb, sb, i, j, q);
    fp_trans<ARC>(G, cb, sb, q, f);
    fp_axial<ARC>(G, q, zs, f.B0, f.H);
}

// Antiderivative of the unit-height trapezoid at column-relative coordinate u
// (SURVEY.md 8c.5), in column units.
__device__ __forceinline__ float trap_T(const Footprint& f, float u) {
    const float p1 = fminf(fmaxf(u, f.u0), f.u1) - f.u0;
    const float fl = fminf(fmaxf(u, f.u1), f.u2) - f.u1;
    const float p2 = f.u3 - fminf(fmaxf(u, f.u2), f.u3);
    return p1 * p1 * f.inv2r1 + fl + (f.halfr2 - p2 * p2 * f.inv2r2);
}

// F1 of column s: mean of the trapezoid over the column.
__device__ __forceinline__ float sf_F1(const Footprint& f, int s) {
    const float e0 = ((float)s - 0.5f) - f.sfc;
    const float e1 = ((float)s + 0.5f) - f.sfc;
    return trap_T(f, e1) - trap_T(f, e0);
}

__device__ __forceinline__ float voxel_b(const Footprint& f, int k) { return fmaf((float)k, f.H, f.B0); }

// L_z(s, t): 3-D path length per unit in-plane length of ray (s, t).
template <bool ARC>
__device__ __forceinline__ float ray_Lz(const DGeom& G, int s, int t) {
    const float th = ((float)t + 0.5f - G.t_c0p) * G.dt;
    if (ARC) {
        return sqrtf(fmaf(th, th, G.dsd * G.dsd)) / G.dsd;
    } else {
        const float sg = ((float)s - G.s_c0) * G.delta;
        const float q = fmaf(sg, sg, G.dsd * G.dsd);
        return sqrtf((q + th * th) / q);
    }
}

}  // namespace ctr
