// zslab.cu — volume-domain (z-slab) decomposition of the solve (SURVEY.md 8e /
// 8f row f1, PAPER.md:470 on communication).  Each rank owns a slab of nz
// planes of x, g, htilde, D_L; every rank holds the full sinograms.  One
// sub-iteration of Algorithm 1:
//   1. x-update of the slab (k_update with one halo plane of x from each
//      neighbour slab, so the 26-neighbour stencil sees across slab faces);
//   2. halo exchange of the new x's boundary planes;
//   3. forward projection of the slab for the subset's views (the slab is a
//      sub-volume geometry: same views, nz and z0 of the slab) -> partial p;
//   4. sum of the partial projections (NCCL all-reduce of V_m nt ns floats,
//      4 R_m bytes instead of the view decomposition's 4 N) and the
//      weighted residual r = L_z w (p - y);
//   5. back-projection onto the slab with the g / htilde epilogue.
// All volume work splits over the ranks.  The same driver runs G slabs in one
// process on one GPU (dist == NULL): step 4 sums the local partials in one
// kernel and step 2 is device copies, which is how the decomposition is
// tested here (one GPU per run).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/ctrecon.h"
#include "kernels.cuh"

namespace ctr {

constexpr int ZS_MAXLOCAL = 8;

struct Partials {
    const float* p[ZS_MAXLOCAL];
    int n;
};

// r[vi][t][s] = L_z(s,t) w (sum_i p_i[vi][t][s] - y) with p_i = L_z A_i x (FWD_PLAIN partials);
// ones (D_L): r = w sum_i p_i with p_i = L_z^2 A_i 1 (FWD_ONES_W partials, w = NULL)
// over the views of vsel (subset from ctl when ctl != nullptr).
template <bool ARC, bool ONES>
__global__ void k_zs_resid(DGeom G, const Ctl* __restrict__ ctl, Views vsel, Partials P, const float* __restrict__ y,
                           const float* __restrict__ w, float* __restrict__ r) {
    const Views V = select_views(ctl, vsel);
    const long long per = (long long)G.nt * G.ns;
    const long long n = (long long)V.count * per;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const int vi = (int)(e / per);
        const int rem = (int)(e % per);
        const int t = rem / G.ns, s = rem % G.ns;
        float p = 0.f;
        for (int i = 0; i < P.n; i++) p += P.p[i][e];
        const long long a = (long long)(V.start + vi * V.stride) * per + rem;
        const float wv = w ? __ldg(&w[a]) : 1.f;
        const float lz = G.dim == 3 ? ray_Lz<ARC>(G, s, t) : 1.f;
        // the ones pass (D_L) gets L_z^2 A1 from FWD_ONES_W: only w is left to apply
        r[e] = ONES ? wv * p : lz * wv * (p - __ldg(&y[a]));
    }
}

static void launch_zs_resid(const DGeom& G, const Ctl* ctl, Views v, int max_count, const Partials& P,
                            const float* y, const float* w, float* r, bool ones, cudaStream_t s) {
    const long long n = (long long)max_count * G.nt * G.ns;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (G.arc) {
        if (ones) k_zs_resid<true, true><<<blocks, 256, 0, s>>>(G, ctl, v, P, y, w, r);
        else k_zs_resid<true, false><<<blocks, 256, 0, s>>>(G, ctl, v, P, y, w, r);
    } else {
        if (ones) k_zs_resid<false, true><<<blocks, 256, 0, s>>>(G, ctl, v, P, y, w, r);
        else k_zs_resid<false, false><<<blocks, 256, 0, s>>>(G, ctl, v, P, y, w, r);
    }
    launches_add(1);
}

}  // namespace ctr

using namespace ctr;

// ------------------------------------------------------------------ helpers shared with api.cu
ct_status ctr_fail(ct_status st, const char* fmt, ...);
const DGeom& ctr_geom_dev(const ct_geom* g);
const float4* ctr_geom_vtab(const ct_geom* g);
const ct_geom_desc& ctr_geom_desc(const ct_geom* g);
int ctr_geom_device(const ct_geom* g);
ncclComm_t ctr_dist_comm(const ct_dist* d);
int ctr_dist_rank(const ct_dist* d);
int ctr_dist_world(const ct_dist* d);
ct_status ctr_make_reg(const ct_geom* g, const ct_reg_desc* r, RegParams& rp);
ct_status ctr_validate_params(const ct_geom* g, const oslalm_params* p);

#define ZS_CUDA(call)                                                                            \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess) return ctr_fail(CT_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)
#define ZS_NCCL(call)                                                                            \
    do {                                                                                         \
        ncclResult_t r_ = (call);                                                                \
        if (r_ != ncclSuccess) return ctr_fail(CT_E_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

extern "C" ct_status ct_zslab_range(const ct_geom* g, int rank, int world, int* z0, int* nz) {
    if (!g || !z0 || !nz) return ctr_fail(CT_E_CONFIG, "ct_zslab_range: NULL argument");
    const int NZ = ctr_geom_dev(g).nz;
    if (world < 1 || rank < 0 || rank >= world || world > NZ)
        return ctr_fail(CT_E_CONFIG, "ct_zslab_range: rank %d / world %d for nz = %d", rank, world, NZ);
    const int a = (int)((long long)rank * NZ / world), b = (int)((long long)(rank + 1) * NZ / world);
    *z0 = a;
    *nz = b - a;
    return CT_OK;
}

// the sub-volume geometry of planes [z0, z0 + nzs) of g (same views and detector)
static DGeom slab_geom(const DGeom& G, int z0, int nzs) {
    DGeom S = G;
    S.nz = nzs;
    S.z0 = G.z0 + (float)z0 * G.dz;
    S.zbot = G.zbot + (float)z0 * G.dz;
    S.ztop = S.zbot + (float)nzs * G.dz;
    S.nvox = S.nxy * nzs;
    return S;
}

namespace {
struct ZsLayout {
    size_t ctl, xa, xb, pfx, part, r, total;
};
size_t al(size_t v) { return (v + 255) & ~(size_t)255; }
ZsLayout zs_layout(const DGeom& S, int vcount, bool with_r) {
    ZsLayout L;
    size_t off = 0;
    L.ctl = off;
    off = al(off + sizeof(Ctl));
    L.xa = off;   // x with one halo plane on each side
    off = al(off + sizeof(float) * (size_t)S.nxy * (S.nz + 2));
    L.xb = off;
    off = al(off + sizeof(float) * (size_t)S.nxy * (S.nz + 2));
    L.pfx = off;
    if (S.dim == 3) off = al(off + sizeof(float2) * (size_t)S.nxy * pfx_stride_of(S));
    L.part = off;
    off = al(off + sizeof(float) * (size_t)vcount * S.nt * S.ns);
    L.r = off;
    if (with_r) off = al(off + sizeof(float) * (size_t)vcount * S.nt * S.ns);
    L.total = off;
    return L;
}

struct Slab {
    DGeom S;
    int rank, z0;
    bool lo, hi;            // neighbours below / above exist
    Ctl* ctl;
    float *xa, *xb;         // interior plane 0 of the extended buffers
    float* pfx;
    float* part;
    char* ws;
};
}  // namespace

extern "C" ct_status oslalm_zslab_workspace_size(const ct_geom* g, const oslalm_params* p, int rank, int world,
                                                 size_t* bytes) {
    if (!g || !p || !bytes) return ctr_fail(CT_E_CONFIG, "oslalm_zslab_workspace_size: NULL argument");
    ct_status st = ctr_validate_params(g, p);
    if (st != CT_OK) return st;
    int z0, nzs;
    st = ct_zslab_range(g, rank, world, &z0, &nzs);
    if (st != CT_OK) return st;
    const DGeom S = slab_geom(ctr_geom_dev(g), z0, nzs);
    const int vcount = std::max((ctr_geom_desc(g).na + p->M - 1) / p->M, 1);
    *bytes = zs_layout(S, vcount, true).total;
    return CT_OK;
}

// the local slabs rank0 .. rank0 + nlocal - 1 of `world`; dist == NULL: all slabs local
static ct_status zs_setup(const ct_geom* g, int nlocal, int world, const ct_dist* dist, int vcount,
                          void* const* workspace, size_t workspace_bytes, std::vector<Slab>& sl) {
    if (nlocal < 1 || nlocal > ZS_MAXLOCAL) return ctr_fail(CT_E_CONFIG, "1 <= local slabs <= %d", ZS_MAXLOCAL);
    if (dist && nlocal != 1) return ctr_fail(CT_E_CONFIG, "with a communicator each process drives one slab");
    if (!dist && nlocal != world) return ctr_fail(CT_E_CONFIG, "without a communicator all %d slabs are local", world);
    const int rank0 = dist ? ctr_dist_rank(dist) : 0;
    if (dist && ctr_dist_world(dist) != world) return ctr_fail(CT_E_CONFIG, "world != communicator size");
    sl.resize(nlocal);
    for (int i = 0; i < nlocal; i++) {
        Slab& s = sl[i];
        s.rank = rank0 + i;
        int z0, nzs;
        ct_status st = ct_zslab_range(g, s.rank, world, &z0, &nzs);
        if (st != CT_OK) return st;
        s.S = slab_geom(ctr_geom_dev(g), z0, nzs);
        s.z0 = z0;
        s.lo = s.rank > 0;
        s.hi = s.rank + 1 < world;
        if (!workspace[i]) return ctr_fail(CT_E_CONFIG, "workspace[%d] is NULL", i);
        const ZsLayout L = zs_layout(s.S, vcount, i == 0);
        if (workspace_bytes < L.total)
            return ctr_fail(CT_E_NOMEM, "workspace %zu < %zu bytes (oslalm_zslab_workspace_size)", workspace_bytes,
                            L.total);
        s.ws = (char*)workspace[i];
        s.ctl = (Ctl*)(s.ws + L.ctl);
        s.xa = (float*)(s.ws + L.xa) + s.S.nxy;
        s.xb = (float*)(s.ws + L.xb) + s.S.nxy;
        s.pfx = s.S.dim == 3 ? (float*)(s.ws + L.pfx) : nullptr;
        s.part = (float*)(s.ws + L.part);
    }
    return CT_OK;
}

// halo planes of buffer `which` (0: xa, 1: xb) of every local slab from its neighbours
static ct_status zs_halo(std::vector<Slab>& sl, int which, const ct_dist* dist, cudaStream_t s) {
    auto buf = [&](Slab& q) { return which ? q.xb : q.xa; };
    if (!dist) {
        for (size_t i = 0; i < sl.size(); i++) {
            Slab& q = sl[i];
            const size_t pl = sizeof(float) * q.S.nxy;
            if (q.lo) {
                Slab& b = sl[i - 1];
                ZS_CUDA(cudaMemcpyAsync(buf(q) - q.S.nxy, buf(b) + (size_t)(b.S.nz - 1) * b.S.nxy, pl,
                                        cudaMemcpyDeviceToDevice, s));
            }
            if (q.hi) {
                Slab& a = sl[i + 1];
                ZS_CUDA(cudaMemcpyAsync(buf(q) + (size_t)q.S.nz * q.S.nxy, buf(a), pl, cudaMemcpyDeviceToDevice, s));
            }
        }
        return CT_OK;
    }
    Slab& q = sl[0];
    ncclComm_t comm = ctr_dist_comm(dist);
    const size_t n = (size_t)q.S.nxy;
    ZS_NCCL(ncclGroupStart());
    if (q.lo) {
        ZS_NCCL(ncclSend(buf(q), n, ncclFloat, q.rank - 1, comm, s));
        ZS_NCCL(ncclRecv(buf(q) - n, n, ncclFloat, q.rank - 1, comm, s));
    }
    if (q.hi) {
        ZS_NCCL(ncclSend(buf(q) + (size_t)(q.S.nz - 1) * n, n, ncclFloat, q.rank + 1, comm, s));
        ZS_NCCL(ncclRecv(buf(q) + (size_t)q.S.nz * n, n, ncclFloat, q.rank + 1, comm, s));
    }
    ZS_NCCL(ncclGroupEnd());
    return CT_OK;
}

// partial projections of every local slab -> residual r in slab 0's workspace (all-reduce with NCCL)
static ct_status zs_reduce_resid(std::vector<Slab>& sl, const DGeom& G, const Ctl* ctl, Views v, int count,
                                 const float* y, const float* w, float* r, bool ones, const ct_dist* dist,
                                 cudaStream_t s) {
    Partials P;
    P.n = (int)sl.size();
    for (size_t i = 0; i < sl.size(); i++) P.p[i] = sl[i].part;
    if (dist) {
        ZS_NCCL(ncclAllReduce(sl[0].part, sl[0].part, (size_t)count * G.nt * G.ns, ncclFloat, ncclSum,
                              ctr_dist_comm(dist), s));
    }
    launch_zs_resid(G, ctl, v, count, P, y, w, r, ones, s);
    return CT_OK;
}

extern "C" ct_status ct_sqs_diag_zslab(const ct_geom* g, const float* w, int nlocal, int world, const ct_dist* dist,
                                       float* const* d_out, void* const* workspace, size_t workspace_bytes,
                                       ct_stream stream) {
    if (!g || !d_out || !workspace) return ctr_fail(CT_E_CONFIG, "ct_sqs_diag_zslab: NULL argument");
    const ct_geom_desc& d = ctr_geom_desc(g);
    // views per pass: as many as the workspace holds (zs_setup validates every local slab)
    int z0, nzs;
    ct_status st0 = ct_zslab_range(g, dist ? ctr_dist_rank(dist) : 0, world, &z0, &nzs);
    if (st0 != CT_OK) return st0;
    const DGeom S0 = slab_geom(ctr_geom_dev(g), z0, nzs + 1);
    int chunk = std::min(d.na, 256);
    while (chunk > 1 && zs_layout(S0, chunk, true).total > workspace_bytes) chunk--;
    std::vector<Slab> sl;
    ct_status st = zs_setup(g, nlocal, world, dist, chunk, workspace, workspace_bytes, sl);
    if (st != CT_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const DGeom& G = ctr_geom_dev(g);
    float* r = (float*)(sl[0].ws + zs_layout(sl[0].S, chunk, true).r);
    for (size_t i = 0; i < sl.size(); i++) ZS_CUDA(cudaMemsetAsync(d_out[i], 0, sizeof(float) * sl[i].S.nvox, s));
    for (int c0 = 0; c0 < d.na; c0 += chunk) {
        const int cnt = std::min(chunk, d.na - c0);
        Views vv{c0, 1, cnt};
        for (auto& q : sl)
            launch_fwd(q.S, ctr_geom_vtab(g), nullptr, vv, cnt, nullptr, nullptr, nullptr, nullptr, q.part, FWD_ONES_W,
                       s);
        // FWD_ONES_W with w = NULL leaves p = L_z A1; the weights and L_z come in the residual
        st = zs_reduce_resid(sl, G, nullptr, vv, cnt, nullptr, w, r, true, dist, s);
        if (st != CT_OK) return st;
        for (size_t i = 0; i < sl.size(); i++)
            launch_back(sl[i].S, ctr_geom_vtab(g), nullptr, vv, r, 1.0f, BK_ACCUM, false, d_out[i], nullptr, nullptr,
                        s);
    }
    ZS_CUDA(cudaGetLastError());
    return CT_OK;
}

extern "C" ct_status oslalm_zslab_solve(const ct_geom* g, const float* y, const float* w, const ct_reg_desc* r,
                                        const float* const* d_l, const oslalm_params* p, oslalm_state* st_, int nlocal,
                                        int world, int n_subiters, const ct_dist* dist, void* const* workspace,
                                        size_t workspace_bytes, ct_stream stream) {
    if (!g || !y || !d_l || !st_ || !workspace || !p) return ctr_fail(CT_E_CONFIG, "oslalm_zslab_solve: NULL argument");
    ct_status st = ctr_validate_params(g, p);
    if (st != CT_OK) return st;
    RegParams rp;
    st = ctr_make_reg(g, r, rp);
    if (st != CT_OK) return st;
    if (n_subiters < 0) return ctr_fail(CT_E_CONFIG, "n_subiters < 0");
    const ct_geom_desc& d = ctr_geom_desc(g);
    const int M = p->M;
    const int vcount = (d.na + M - 1) / M;
    std::vector<Slab> sl;
    st = zs_setup(g, nlocal, world, dist, vcount, workspace, workspace_bytes, sl);
    if (st != CT_OK) return st;
    const long long k0 = st_[0].k;
    for (int i = 0; i < nlocal; i++) {
        if (!st_[i].x || !st_[i].g || !st_[i].htilde || !d_l[i]) return ctr_fail(CT_E_CONFIG, "slab %d: NULL state", i);
        if (st_[i].k != k0) return ctr_fail(CT_E_CONFIG, "slab states disagree on k");
    }
    cudaStream_t s = (cudaStream_t)stream;
    const DGeom& G = ctr_geom_dev(g);
    const float4* vtab = ctr_geom_vtab(g);
    float* rbuf = (float*)(sl[0].ws + zs_layout(sl[0].S, vcount, true).r);
    const float lo = (float)p->box_lo, hi = std::isinf(p->box_hi) ? 3.0e38f : (float)p->box_hi;
    for (int i = 0; i < nlocal; i++) {
        Ctl h;
        memset(&h, 0, sizeof(h));
        h.k = k0;
        h.k_base = k0;
        h.M = M;
        h.na = d.na;
        h.rank = 0;   // every slab projects all views of the subset
        h.world = 1;
        h.rho_fixed_mode = p->rho_mode == OSLALM_RHO_FIXED;
        h.simple = p->variant == OSLALM_SIMPLE;
        h.alpha = (float)p->alpha;
        h.rho_fixed = (float)p->rho_fixed;
        ZS_CUDA(cudaMemcpyAsync(sl[i].ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, s));
        ZS_CUDA(cudaMemcpyAsync(sl[i].xa, st_[i].x, sizeof(float) * sl[i].S.nvox, cudaMemcpyDeviceToDevice, s));
    }
    st = zs_halo(sl, 0, dist, s);
    if (st != CT_OK) return st;
    // line 1 (k == 0): rho = 1, zeta = g = M grad L_{M-1}(x) (or the full gradient), htilde = zeta
    if (k0 == 0) {
        const bool full = p->init_grad == OSLALM_INIT_FULL;
        const int m = M - 1;
        const int cnt_last = (d.na - m + M - 1) / M;
        for (int c0 = 0; c0 < (full ? d.na : 1); c0 += vcount) {
            Views vv = full ? Views{c0, 1, std::min(vcount, d.na - c0)} : Views{m, M, cnt_last};
            if (vv.count <= 0) continue;
            for (auto& q : sl)
                launch_fwd(q.S, vtab, nullptr, vv, vv.count, q.xa, q.xa, nullptr, nullptr, q.part, FWD_PLAIN, s);
            st = zs_reduce_resid(sl, G, nullptr, vv, vv.count, y, w, rbuf, false, dist, s);
            if (st != CT_OK) return st;
            for (int i = 0; i < nlocal; i++) {
                if (full)
                    launch_back(sl[i].S, vtab, nullptr, vv, rbuf, 1.0f, c0 == 0 ? BK_WRITE : BK_ACCUM, false,
                                st_[i].g, nullptr, nullptr, s);
                else
                    launch_back(sl[i].S, vtab, nullptr, vv, rbuf, (float)M, BK_INIT, false, nullptr, st_[i].g,
                                st_[i].htilde, s);
            }
        }
        if (full)
            for (int i = 0; i < nlocal; i++)
                launch_init_from_zeta(sl[i].S, st_[i].g, st_[i].g, st_[i].htilde, s);
    }
    // sub-iterations (eager; the kernels select the subset and rho from Ctl.k)
    for (int it = 0; it < n_subiters; it++) {
        const int cur = it & 1;   // buffer holding x: 0 = xa, 1 = xb (k_update reads by the same parity)
        for (int i = 0; i < nlocal; i++) {
            Slab& q = sl[i];
            launch_update_halo(q.S, rp, q.ctl, q.xa, q.xb, d_l[i], st_[i].g, st_[i].htilde, lo, hi, q.pfx, q.lo,
                               q.hi, s);
        }
        st = zs_halo(sl, cur ^ 1, dist, s);
        if (st != CT_OK) return st;
        for (auto& q : sl) {
            if (q.pfx)   // 3-D: the forward resamples the slab's z-prefix written by the update
                launch_fwd(q.S, vtab, q.ctl, Views{0, 1, 0}, vcount, q.pfx, q.pfx, nullptr, nullptr, q.part, FWD_PLAIN,
                           s, pfx_stride_of(q.S));
            else         // 2-D: reads the new x (buffer by the parity of k - k_base, as the update wrote it)
                launch_fwd(q.S, vtab, q.ctl, Views{0, 1, 0}, vcount, q.xa, q.xb, nullptr, nullptr, q.part, FWD_PLAIN, s);
        }
        st = zs_reduce_resid(sl, G, sl[0].ctl, Views{0, 1, 0}, vcount, y, w, rbuf, false, dist, s);
        if (st != CT_OK) return st;
        for (int i = 0; i < nlocal; i++) {
            launch_back(sl[i].S, vtab, sl[i].ctl, Views{0, 1, 0}, rbuf, (float)M, BK_UPDATE, false, nullptr, st_[i].g,
                        st_[i].htilde, s);   // its last block advances k
        }
    }
    const int fin = n_subiters & 1;
    for (int i = 0; i < nlocal; i++) {
        ZS_CUDA(cudaMemcpyAsync(st_[i].x, fin ? sl[i].xb : sl[i].xa, sizeof(float) * sl[i].S.nvox,
                                cudaMemcpyDeviceToDevice, s));
        st_[i].k = k0 + n_subiters;
    }
    ZS_CUDA(cudaGetLastError());
    return CT_OK;
}
