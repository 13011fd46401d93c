// api.cu — the extern "C" boundary of libctrecon.so (include/ctrecon.h):
// argument validation (before any launch), geometry handle, projector /
// regulariser entry points, the Algorithm 1 solver with its CUDA-graph replay
// and the NCCL view-sharded path.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ctrecon.h"
#include "kernels.cuh"

using namespace ctr;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

namespace ctr {
int64_t launches_add(int64_t n) { return g_launches.fetch_add(n) + n; }
thread_local bool g_pdl = false;
#ifndef CTR_PDL
#define CTR_PDL 1   // programmatic dependent launch inside the solve's sub-iteration graph
#endif

// programmatic dependent launches for the kernels enqueued in this scope (kernels.cuh)
struct PdlScope {
    bool old;
    explicit PdlScope(bool on) : old(g_pdl) { g_pdl = on; }
    ~PdlScope() { g_pdl = old; }
};
}  // namespace ctr

static ct_status fail(ct_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CT_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return fail(CT_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define CT_NCCL(call)                                                                        \
    do {                                                                                     \
        ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess) return fail(CT_E_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

// NVTX range for the duration of a scope (profiler timelines; no cost without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ handles
struct GraphKey {
    std::vector<uintptr_t> ptrs;
    std::vector<double> vals;
    bool operator<(const GraphKey& o) const { return std::tie(ptrs, vals) < std::tie(o.ptrs, o.vals); }
};

// Schedule of the segmented forward for one (view stride, view count) (launch_fwd_seg).
struct SegSched {
    int2* d = nullptr;   // device entries (vi, block | segment << 16)
    int n = 0, seg_len = 0, nseg = 0;
};

struct ct_geom {
    ct_geom_desc d;
    DGeom G;
    int device;
    float4* vtab;             // per view: cos beta, sin beta, z_s, 0
    std::vector<float4> htab; // host copy (segmented-forward schedules)
    int fwd_nseg = -1;        // ct_geom_set_fwd_segments: -1 automatic, 0 off, >= 2 forced
    cudaStream_t cap_stream;  // private stream for graph capture
    std::mutex mu;            // guards the graph and schedule caches (the geometry itself is immutable)
    std::map<GraphKey, cudaGraphExec_t> graphs;
    std::map<std::tuple<int, int, int>, SegSched> seg;   // (view stride, views, segments)
};

// Segments of the z-prefix forward of `views` views per launch (0 = unsegmented).
// Automatic: 16 when the z-prefix array exceeds 512 MB (c5: 2.2 GB; every view would otherwise
// re-stream its band of it from HBM); for volumes of at least 256 x 256 columns, as many as keep
// the partial sums within 96 MB (at most 8; measured optimum c4: 3, c3: 8, profiles/r2s/
// nseg_sweep.log: the tile-ordered walk's L2 hit rate against the partials' traffic); otherwise
// none (small volumes, 2-D).
static int fwd_nseg_of(const ct_geom* g, long long views) {
    if (g->G.dim != 3) return 0;
    if (g->fwd_nseg >= 0) return g->fwd_nseg >= 2 ? g->fwd_nseg : 0;
    const double pfx = 8.0 * (double)g->G.nxy * (double)pfx_stride_of(g->G);
    if (pfx > 512.0 * 1024.0 * 1024.0) return 16;
    if (g->G.nxy < 256LL * 256LL || views < 1) return 0;
    const double per = 4.0 * (double)views * g->G.nt * g->G.ns;
    const int n = (int)std::min(8.0, std::floor(96.0 * 1024.0 * 1024.0 / per));
    return n >= 2 ? n : 0;
}

// floats of the segmented forward's partial buffer for up to `count` views (0 = unsegmented)
static size_t fwd_part_floats(const ct_geom* g, long long count) {
    const int ns = fwd_nseg_of(g, count);
    return ns ? (size_t)ns * (size_t)count * g->G.nt * g->G.ns : 0;
}

struct ct_dist {
    ncclComm_t comm;                // NULL for a local (single-process) emulation
    int rank, world, device;
    cudaStream_t side;              // high-priority stream: stencil of the new x during the reduction
    cudaEvent_t ev_x, ev_sten;      // x+ written / stencil done
    bool local;                     // ct_dist_create_local: this process plays all `world` ranks
};

// Owner slab of rank q of W (the plane range of ct_zslab_range): 3-D volumes split their z-planes;
// 2-D images are not split (every rank owns the whole image and the partial gradients are
// all-reduced instead of reduce-scattered).
static void owner_slab(const DGeom& G, int q, int W, int* z0, int* nz) {
    if (G.dim != 3) {
        *z0 = 0;
        *nz = G.nz;
        return;
    }
    const int a = (int)((long long)q * G.nz / W), b = (int)((long long)(q + 1) * G.nz / W);
    *z0 = a;
    *nz = b - a;
}

// local ranks whose work this process runs (all of them in a local emulation)
static int local_ranks(const ct_dist* dist) { return dist && dist->local ? dist->world : 1; }

static DGeom sub_geom(const DGeom& G, int z0, int nzs) {
    DGeom S = G;
    S.nz = nzs;
    S.z0 = G.z0 + (float)z0 * G.dz;
    S.zbot = G.zbot + (float)z0 * G.dz;
    S.ztop = S.zbot + (float)nzs * G.dz;
    S.nvox = S.nxy * nzs;
    return S;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

static ct_status check_async() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(CT_E_CUDA, "CUDA launch/async error: %s", cudaGetErrorString(e));
    return CT_OK;
}

static size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

// ------------------------------------------------------------------ geometry
static ct_status validate_desc(const ct_geom_desc* d) {
    if (!d) return fail(CT_E_CONFIG, "ct_geom_desc is NULL");
    if (d->dim != 2 && d->dim != 3) return fail(CT_E_CONFIG, "dim must be 2 or 3 (got %d)", d->dim);
    if (d->nx <= 0 || d->ny <= 0 || d->nz <= 0 || d->ns <= 0 || d->nt <= 0 || d->na <= 0)
        return fail(CT_E_CONFIG, "sizes must be positive");
    if (d->dim == 2 && (d->nz != 1 || d->nt != 1)) return fail(CT_E_CONFIG, "2-D geometry needs nz = nt = 1");
    if (!(d->dx > 0 && d->dy > 0 && d->dz > 0 && d->ds > 0 && d->dt > 0))
        return fail(CT_E_CONFIG, "spacings must be positive");
    if (!(d->dso > 0 && d->dsd > d->dso)) return fail(CT_E_CONFIG, "need 0 < dso < dsd");
    if (d->det_shape != CT_DET_FLAT && d->det_shape != CT_DET_ARC) return fail(CT_E_CONFIG, "bad det_shape");
    if (!std::isfinite(d->orbit_deg) || !std::isfinite(d->orbit_start_deg) || !std::isfinite(d->pitch) ||
        !std::isfinite(d->source_z0))
        return fail(CT_E_CONFIG, "non-finite orbit parameters");
    if ((long long)d->nx * d->ny * d->nz >= (1LL << 32)) return fail(CT_E_CONFIG, "volume of 2^32 voxels or more");
    // the 3-D forward addresses the z-prefix array (nx ny columns of round2(nz + 2) float2 entries)
    // with 32-bit element offsets, and voxel columns j nx + i in int
    if (d->dim == 3 && (long long)d->nx * d->ny * (((long long)d->nz + 2) & ~1LL) >= (1LL << 32))
        return fail(CT_E_CONFIG, "z-prefix array of nx*ny*(nz+2) >= 2^32 entries");
    if (d->nt > 128) return fail(CT_E_CONFIG, "nt = %d > 128 detector rows", d->nt);
    // the 3-D forward's candidate list packs a voxel column (i, j) into 16 + 16 bits
    if (d->dim == 3 && (d->nx > 65535 || d->ny > 65535))
        return fail(CT_E_CONFIG, "nx = %d, ny = %d: at most 65535 columns per axis in 3-D", d->nx, d->ny);
    // the update kernel keeps x+ of a 32-column tile in shared memory for the z-prefix
    if (d->nz > 1536) return fail(CT_E_CONFIG, "nz = %d > 1536 slices", d->nz);
    // source must stay outside the volume's circumscribed cylinder
    const double ex = 0.5 * d->nx * d->dx + std::fabs(d->offset_x);
    const double ey = 0.5 * d->ny * d->dy + std::fabs(d->offset_y);
    const double rmax = std::sqrt(ex * ex + ey * ey);
    if (rmax >= 0.95 * d->dso) return fail(CT_E_CONFIG, "volume reaches the source circle");
    // footprint width bound (columns) for the back-projector's per-thread slots
    const double dmin = d->dso - rmax;
    const double diag = std::sqrt(d->dx * d->dx + d->dy * d->dy);
    double width;
    if (d->det_shape == CT_DET_ARC) {
        width = 2.0 * std::asin(std::min(1.0, 0.5 * diag / dmin)) / (d->ds / d->dsd);
    } else {
        const double th = std::asin(rmax / d->dso);
        const double c = std::cos(th);
        width = d->dsd * (diag / dmin) / (c * c) / d->ds;
    }
    // corner-offset angle seen from the source (small-angle atan in ct_footprint)
    if (0.5 * diag / dmin > 0.05) return fail(CT_E_CONFIG, "voxels too large for their distance to the source");
    if (width + 2.0 > kMaxCells)
        return fail(CT_E_CONFIG, "voxel footprint spans up to %.1f detector columns (limit %d)", width + 2.0,
                    kMaxCells);
    return CT_OK;
}

static DGeom make_dgeom(const ct_geom_desc* d) {
    DGeom G;
    G.dim = d->dim;
    G.nx = d->nx;
    G.ny = d->ny;
    G.nz = d->dim == 3 ? d->nz : 1;
    G.ns = d->ns;
    G.nt = d->dim == 3 ? d->nt : 1;
    G.arc = d->det_shape == CT_DET_ARC;
    G.na = d->na;
    G.dx = (float)d->dx;
    G.dy = (float)d->dy;
    G.dz = (float)d->dz;
    G.x0 = (float)(-0.5 * (d->nx - 1) * d->dx + d->offset_x);
    G.y0 = (float)(-0.5 * (d->ny - 1) * d->dy + d->offset_y);
    G.z0 = (float)(-0.5 * (G.nz - 1) * d->dz + d->offset_z);
    const double delta = G.arc ? d->ds / d->dsd : d->ds;
    G.delta = (float)delta;
    G.inv_delta = (float)(1.0 / delta);
    G.s_c0 = (float)(0.5 * (d->ns - 1) + d->offset_s);
    G.t_c0p = (float)(0.5 * (G.nt - 1) + d->offset_t + 0.5);
    G.dt = (float)d->dt;
    G.inv_dt = (float)(1.0 / d->dt);
    G.dso = (float)d->dso;
    G.dsd = (float)d->dsd;
    G.zbot = (float)(-0.5 * G.nz * d->dz + d->offset_z);
    G.ztop = (float)(0.5 * G.nz * d->dz + d->offset_z);
    {
        const double ex = 0.5 * d->nx * d->dx + std::fabs(d->offset_x);
        const double ey = 0.5 * d->ny * d->dy + std::fabs(d->offset_y);
        G.rxy = (float)(std::sqrt(ex * ex + ey * ey) * (1.0 + 1e-6));
    }
    G.zs0 = (float)(d->dim == 3 ? d->source_z0 : 0.0);
    G.zstep = (float)(d->dim == 3 ? d->pitch * d->nt * d->dt * d->dso / d->dsd * (d->orbit_deg / 360.0) / d->na : 0.0);
    G.nxy = (long long)d->nx * d->ny;
    G.nvox = G.nxy * G.nz;
    return G;
}

extern "C" ct_status ct_geom_create(const ct_geom_desc* d, int device, ct_geom** out) {
    if (!out) return fail(CT_E_CONFIG, "out is NULL");
    *out = nullptr;
    ct_status st = validate_desc(d);
    if (st != CT_OK) return st;
    int ndev = 0;
    CT_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CT_E_CONFIG, "device %d not present (%d devices)", device, ndev);
    DeviceGuard guard(device);
    std::vector<float4> tab(d->na);
    const double pi = 3.14159265358979323846;
    const double zstep = d->pitch * d->nt * d->dt * d->dso / d->dsd * (d->orbit_deg / 360.0) / d->na;
    for (int v = 0; v < d->na; v++) {
        const double beta = d->orbit_start_deg * pi / 180.0 + (d->orbit_deg * pi / 180.0) * v / d->na;
        tab[v] = make_float4((float)std::cos(beta), (float)std::sin(beta),
                             (float)(d->dim == 3 ? d->source_z0 + v * zstep : 0.0), 0.f);
    }
    ct_geom* g = new ct_geom();
    g->d = *d;
    g->htab = tab;
    g->G = make_dgeom(d);
    g->device = device;
    g->vtab = nullptr;
    cudaError_t e = cudaMalloc(&g->vtab, sizeof(float4) * d->na);
    if (e == cudaSuccess) e = cudaMemcpy(g->vtab, tab.data(), sizeof(float4) * d->na, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        if (g->vtab) cudaFree(g->vtab);
        delete g;
        return fail(CT_E_CUDA, "ct_geom_create: %s", cudaGetErrorString(e));
    }
    *out = g;
    return CT_OK;
}

extern "C" void ct_geom_destroy(ct_geom* g) {
    if (!g) return;
    DeviceGuard guard(g->device);
    for (auto& kv : g->graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : g->seg) cudaFree(kv.second.d);
    cudaStreamDestroy(g->cap_stream);
    cudaFree(g->vtab);
    delete g;
}

static ct_status check_views(const ct_geom* g, ct_views v) {
    if (v.count < 0) return fail(CT_E_SHAPE, "view count %d < 0", v.count);
    if (v.count == 0) return CT_OK;
    if (v.stride < 1) return fail(CT_E_SHAPE, "view stride must be >= 1");
    const long long last = (long long)v.start + (long long)(v.count - 1) * v.stride;
    if (v.start < 0 || last >= g->d.na)
        return fail(CT_E_SHAPE, "views {%d,%d,%d} outside [0, %d)", v.start, v.stride, v.count, g->d.na);
    if (v.count > 65535) return fail(CT_E_SHAPE, "at most 65535 views per call (got %d)", v.count);
    if ((long long)v.count * g->G.nt * g->G.ns >= (1LL << 31))
        return fail(CT_E_SHAPE, "projection block of %d views exceeds 2^31 elements", v.count);
    return CT_OK;
}

static Views to_views(ct_views v) { return Views{v.start, v.stride, v.count}; }

// The segmented forward's schedule for views of stride `stride` (angles of start 0; the order is
// a locality heuristic only), built and uploaded on first use -- never inside a graph capture
// (solve_impl and ct_forward_zprefix build it before enqueueing).
static ct_status seg_sched(const ct_geom* g, int stride, int count, int nseg, const SegSched** out) {
    ct_geom* gm = const_cast<ct_geom*>(g);
    std::lock_guard<std::mutex> lk(gm->mu);
    const auto key = std::make_tuple(stride, count, nseg);
    auto it = gm->seg.find(key);
    if (it == gm->seg.end()) {
        SegSched S;
        std::vector<int2> h = fwd_seg_schedule(g->G, g->htab, Views{0, stride, count}, count, nseg, &S.seg_len);
        S.n = (int)h.size();
        S.nseg = (std::max(g->G.nx, g->G.ny) + S.seg_len - 1) / S.seg_len;
        CT_CUDA(cudaMalloc(&S.d, sizeof(int2) * h.size()));
        CT_CUDA(cudaMemcpy(S.d, h.data(), sizeof(int2) * h.size(), cudaMemcpyHostToDevice));
        it = gm->seg.emplace(key, S).first;
    }
    *out = &it->second;
    return CT_OK;
}

// z-prefix forward of `max_count` views (from ctl, or v), segmented when S != nullptr (S from
// seg_sched, obtained before any graph capture; part: fwd_part_floats(g, max_count) floats).
static void fwd_pfx(const ct_geom* g, const Ctl* ctl, Views v, const SegSched* S, int max_count, const float* xt,
                    const float* y, const float* w, float* out, int mode, float* part, cudaStream_t s) {
    if (S) {
        launch_fwd_seg(g->G, g->vtab, ctl, v, max_count, xt, y, w, out, mode, s, pfx_stride_of(g->G), S->d, S->n,
                       S->seg_len, S->nseg, part);
    } else {
        launch_fwd(g->G, g->vtab, ctl, v, max_count, xt, xt, y, w, out, mode, s, pfx_stride_of(g->G));
    }
}

extern "C" ct_status ct_geom_set_fwd_segments(ct_geom* g, int nseg) {
    if (!g) return fail(CT_E_CONFIG, "ct_geom_set_fwd_segments: NULL geometry");
    if (nseg < -1 || nseg > 64) return fail(CT_E_CONFIG, "nseg = %d outside [-1, 64]", nseg);
    std::lock_guard<std::mutex> lk(g->mu);
    g->fwd_nseg = nseg;
    DeviceGuard guard(g->device);
    cudaDeviceSynchronize();   // no launch may still read a schedule or graph freed below
    for (auto& kv : g->graphs) cudaGraphExecDestroy(kv.second);
    g->graphs.clear();
    for (auto& kv : g->seg) cudaFree(kv.second.d);
    g->seg.clear();
    return CT_OK;
}

extern "C" ct_status ct_geom_fwd_segments(const ct_geom* g, int views, int* nseg) {
    if (!g || !nseg) return fail(CT_E_CONFIG, "ct_geom_fwd_segments: NULL argument");
    *nseg = fwd_nseg_of(g, views);
    return CT_OK;
}

// ------------------------------------------------------------------ projector
extern "C" ct_status ct_forward(const ct_geom* g, const float* x, ct_views v, float* proj, ct_stream s) {
    if (!g || !x || !proj) return fail(CT_E_CONFIG, "ct_forward: NULL argument");
    ct_status st = check_views(g, v);
    if (st != CT_OK) return st;
    DeviceGuard guard(g->device);
    launch_fwd(g->G, g->vtab, nullptr, to_views(v), v.count, x, x, nullptr, nullptr, proj, FWD_PLAIN,
               (cudaStream_t)s);
    return check_async();
}

// views per launch of a segmented ct_forward_zprefix (its partial buffer is sized for these)
constexpr int kZpfxChunk = 128;

static size_t zprefix_bytes(const ct_geom* g) {
    return g->G.dim == 3 ? align_up(sizeof(float2) * (size_t)g->G.nxy * pfx_stride_of(g->G)) : 0;
}

extern "C" ct_status ct_zprefix_size(const ct_geom* g, size_t* bytes) {
    if (!g || !bytes) return fail(CT_E_CONFIG, "ct_zprefix_size: NULL argument");
    *bytes = g->G.dim == 3 ? zprefix_bytes(g) + sizeof(float) * fwd_part_floats(g, std::min(kZpfxChunk, g->d.na)) : 0;
    return CT_OK;
}

extern "C" ct_status ct_forward_zprefix(const ct_geom* g, const float* x, ct_views v, float* proj, void* workspace,
                                        size_t workspace_bytes, ct_stream s) {
    if (!g || !x || !proj) return fail(CT_E_CONFIG, "ct_forward_zprefix: NULL argument");
    ct_status st = check_views(g, v);
    if (st != CT_OK) return st;
    if (g->G.dim != 3) return ct_forward(g, x, v, proj, s);
    size_t need = 0;
    ct_zprefix_size(g, &need);
    if (!workspace || workspace_bytes < need)
        return fail(CT_E_NOMEM, "ct_forward_zprefix: workspace %zu < %zu bytes", workspace_bytes, need);
    if ((uintptr_t)workspace % 16) return fail(CT_E_CONFIG, "ct_forward_zprefix: workspace not 16-byte aligned");
    DeviceGuard guard(g->device);
    float* pfx = (float*)workspace;
    launch_zprefix(g->G, x, pfx, (cudaStream_t)s);
    // one segment count for every chunk of this call (the partial buffer is sized for it)
    const int nseg = fwd_nseg_of(g, std::min(kZpfxChunk, g->d.na));
    if (!nseg) {
        launch_fwd(g->G, g->vtab, nullptr, to_views(v), v.count, pfx, pfx, nullptr, nullptr, proj, FWD_PLAIN,
                   (cudaStream_t)s, pfx_stride_of(g->G));
        return check_async();
    }
    // segmented: chunks of kZpfxChunk views through the partial buffer after the z-prefix
    float* part = (float*)((char*)workspace + zprefix_bytes(g));
    for (int c0 = 0; c0 < v.count; c0 += kZpfxChunk) {
        const int cnt = std::min(kZpfxChunk, v.count - c0);
        const SegSched* S;
        st = seg_sched(g, v.stride, cnt, nseg, &S);
        if (st != CT_OK) return st;
        fwd_pfx(g, nullptr, Views{v.start + c0 * v.stride, v.stride, cnt}, S, cnt, pfx, nullptr, nullptr,
                proj + (size_t)c0 * g->G.nt * g->G.ns, FWD_PLAIN, part, (cudaStream_t)s);
    }
    return check_async();
}

extern "C" ct_status ct_back(const ct_geom* g, const float* proj, ct_views v, float scale, int accumulate,
                             float* x_out, ct_stream s) {
    if (!g || !proj || !x_out) return fail(CT_E_CONFIG, "ct_back: NULL argument");
    ct_status st = check_views(g, v);
    if (st != CT_OK) return st;
    DeviceGuard guard(g->device);
    launch_back(g->G, g->vtab, nullptr, to_views(v), proj, scale, accumulate ? BK_ACCUM : BK_WRITE,
                g->G.dim == 3, x_out, nullptr, nullptr, (cudaStream_t)s);
    return check_async();
}

extern "C" ct_status ct_sqs_diag(const ct_geom* g, const float* w, const ct_dist* dist, float* d_out,
                                 void* workspace, size_t workspace_bytes, ct_stream s) {
    if (!g || !d_out || !workspace) return fail(CT_E_CONFIG, "ct_sqs_diag: NULL argument");
    const size_t per_view = (size_t)g->G.nt * g->G.ns * sizeof(float);
    int chunk = (int)std::min<size_t>(workspace_bytes / per_view, 65535);
    if (chunk < 1) return fail(CT_E_NOMEM, "ct_sqs_diag: workspace %zu < %zu bytes", workspace_bytes, per_view);
    DeviceGuard guard(g->device);
    NvtxRange nv("ct_sqs_diag");
    cudaStream_t cs = (cudaStream_t)s;
    const int world = dist ? dist->world : 1;
    CT_CUDA(cudaMemsetAsync(d_out, 0, sizeof(float) * g->G.nvox, cs));
    // this rank's views: rank, rank + world, ... (a local emulation runs every rank's share in turn)
    const int q0 = dist && !dist->local ? dist->rank : 0, q1 = dist && !dist->local ? q0 + 1 : local_ranks(dist);
    float* r = (float*)workspace;
    for (int rank = q0; rank < q1; rank++) {
        const int mine = (g->d.na - rank + world - 1) / world;
        for (int c0 = 0; c0 < mine; c0 += chunk) {
            const int cnt = std::min(chunk, mine - c0);
            Views vv{rank + c0 * world, world, cnt};
            launch_fwd(g->G, g->vtab, nullptr, vv, cnt, nullptr, nullptr, nullptr, w, r, FWD_ONES_W, cs);
            launch_back(g->G, g->vtab, nullptr, vv, r, 1.0f, BK_ACCUM, false, d_out, nullptr, nullptr, cs);
        }
    }
    ct_status st = check_async();
    if (st != CT_OK) return st;
    if (dist && !dist->local)
        CT_NCCL(ncclAllReduce(d_out, d_out, (size_t)g->G.nvox, ncclFloat, ncclSum, dist->comm, cs));
    return CT_OK;
}

extern "C" ct_status ct_fbp(const ct_geom* g, const float* proj, float* x_out, void* workspace,
                            size_t workspace_bytes, ct_stream s) {
    if (!g || !proj || !x_out || !workspace) return fail(CT_E_CONFIG, "ct_fbp: NULL argument");
    if (std::fabs(g->d.orbit_deg - 360.0) > 1e-9) return fail(CT_E_CONFIG, "ct_fbp: needs a 360-degree orbit");
    if (g->G.dim == 3 && g->d.pitch != 0.0) return fail(CT_E_CONFIG, "ct_fbp: helical scans are not supported");
    if (g->d.ns > 18000) return fail(CT_E_CONFIG, "ct_fbp: ns > 18000");
    const size_t need = sizeof(float) * (size_t)g->d.na * g->G.nt * g->G.ns;
    if (workspace_bytes < need) return fail(CT_E_NOMEM, "ct_fbp: workspace %zu < %zu bytes", workspace_bytes, need);
    DeviceGuard guard(g->device);
    launch_fbp(g->G, g->vtab, proj, (float*)workspace, x_out, g->d.dsd, (cudaStream_t)s);
    return check_async();
}

extern "C" ct_status ct_kappa_weights(const ct_geom* g, const float* w, float* kappa_out, void* workspace,
                                      size_t workspace_bytes, ct_stream s) {
    if (!g || !kappa_out || !workspace) return fail(CT_E_CONFIG, "ct_kappa_weights: NULL argument");
    const size_t vol = align_up(sizeof(float) * (size_t)g->G.nvox);
    const size_t per_view = (size_t)g->G.nt * g->G.ns * sizeof(float);
    if (workspace_bytes < vol + per_view)
        return fail(CT_E_NOMEM, "ct_kappa_weights: workspace %zu < %zu bytes", workspace_bytes, vol + per_view);
    DeviceGuard guard(g->device);
    cudaStream_t cs = (cudaStream_t)s;
    float* aone = (float*)workspace;                      // A'1
    float* ones = (float*)((char*)workspace + vol);       // a chunk of all-ones views
    const int chunk = (int)std::min<size_t>((workspace_bytes - vol) / per_view, 65535);
    const long long nproj = (long long)chunk * g->G.nt * g->G.ns;
    launch_fill(ones, nproj, 1.f, cs);
    CT_CUDA(cudaMemsetAsync(aone, 0, sizeof(float) * g->G.nvox, cs));
    CT_CUDA(cudaMemsetAsync(kappa_out, 0, sizeof(float) * g->G.nvox, cs));
    const size_t view_elems = (size_t)g->G.nt * g->G.ns;
    for (int c0 = 0; c0 < g->d.na; c0 += chunk) {
        const int cnt = std::min(chunk, g->d.na - c0);
        Views vv{c0, 1, cnt};
        launch_back(g->G, g->vtab, nullptr, vv, ones, 1.0f, BK_ACCUM, g->G.dim == 3, aone, nullptr, nullptr, cs);
        launch_back(g->G, g->vtab, nullptr, vv, w ? w + (size_t)c0 * view_elems : ones, 1.0f, BK_ACCUM,
                    g->G.dim == 3, kappa_out, nullptr, nullptr, cs);     // A'W1 (W1 = w)
    }
    launch_kappa_ratio(g->G.nvox, kappa_out, aone, kappa_out, cs);
    return check_async();
}

static ct_status make_reg(const ct_geom* g, const ct_reg_desc* r, RegParams& rp) {
    if (!r) return fail(CT_E_CONFIG, "ct_reg_desc is NULL");
    if (r->potential < 0 || r->potential > 3) return fail(CT_E_CONFIG, "bad potential %d", r->potential);
    if (r->curvature != CT_CURV_HUBER && r->curvature != CT_CURV_MAX) return fail(CT_E_CONFIG, "bad curvature");
    if (r->potential == CT_POT_QGGMRF && !(r->q >= 1.0 && r->q <= 2.0))
        return fail(CT_E_CONFIG, "q-GGMRF needs 1 <= q <= 2 (got %g)", r->q);
    if (!(r->delta > 0)) return fail(CT_E_CONFIG, "delta must be > 0");
    if (!(r->delta >= 1e-18)) return fail(CT_E_CONFIG, "delta %g below 1e-18 (delta^2 must be a normal float)", r->delta);
    if (r->n_dirs != 4 && r->n_dirs != 13) return fail(CT_E_CONFIG, "n_dirs must be 4 or 13");
    if (g->G.dim == 2 && r->n_dirs != 4) return fail(CT_E_CONFIG, "2-D geometry uses n_dirs = 4");
    for (int i = 0; i < 13; i++) {
        if (!(r->beta[i] >= 0) || !std::isfinite(r->beta[i])) return fail(CT_E_CONFIG, "beta[%d] must be >= 0", i);
        rp.beta[i] = i < r->n_dirs ? (float)r->beta[i] : 0.f;
    }
    rp.delta = (float)r->delta;
    rp.inv_delta = (float)(1.0 / r->delta);
    rp.delta2 = (float)(r->delta * r->delta);
    rp.potential = r->potential;
    rp.n_dirs = r->n_dirs;
    rp.maxcurv = r->curvature == CT_CURV_MAX;
    double bs = 0.0;
    for (int i = 0; i < r->n_dirs; i++) bs += 2.0 * r->beta[i];
    rp.bsum = (float)bs;
    rp.q = (float)(r->potential == CT_POT_QGGMRF ? r->q : 2.0);
    rp.qexp = 2.f - rp.q;
    return CT_OK;
}

extern "C" ct_status ct_reg_grad(const ct_geom* g, const ct_reg_desc* r, const float* x, const float* kappa,
                                 float* grad, float* curv, ct_stream s) {
    if (!g || !x || !grad) return fail(CT_E_CONFIG, "ct_reg_grad: NULL argument");
    RegParams rp;
    ct_status st = make_reg(g, r, rp);
    if (st != CT_OK) return st;
    DeviceGuard guard(g->device);
    launch_reg(g->G, rp, x, kappa, grad, curv, (cudaStream_t)s);
    return check_async();
}

// ------------------------------------------------------------------ solver
struct WsLayout {
    size_t ctl, xalt, xt, part, r, r_stride, zeta, zeta_stride, gradr, curvr, flag, dsum, total;
};


static WsLayout ws_layout(const ct_geom* g, const oslalm_params* p, const ct_dist* dist) {
    const int world = dist ? dist->world : 1;
    const int nl = local_ranks(dist);
    const long long vm = (g->d.na + p->M - 1) / p->M;
    const long long vrank = (vm + world - 1) / world;
    WsLayout L;
    size_t off = 0;
    L.ctl = off;   // one control block per local rank (view selection differs by rank)
    off = align_up(off + sizeof(Ctl) * nl);
    L.xalt = off;
    off = align_up(off + sizeof(float) * g->G.nvox);
    L.xt = off;  // z-prefix array of x+ for the 3-D forward projector
    if (g->G.dim == 3) off = align_up(off + sizeof(float2) * (size_t)g->G.nxy * pfx_stride_of(g->G));
    L.part = off;  // segmented forward: raw segment sums of one rank's views (fwd_part_floats)
    off = align_up(off + sizeof(float) * fwd_part_floats(g, vrank));
    L.r = off;     // residual of each local rank's views
    L.r_stride = align_up(sizeof(float) * (size_t)vrank * g->G.nt * g->G.ns);
    off += L.r_stride * nl;
    L.zeta = off;  // partial back-projection of each local rank (summed in place into the first)
    L.zeta_stride = align_up(sizeof(float) * g->G.nvox);
    if (dist) off += L.zeta_stride * nl;
    L.gradr = off;  // multi-GPU: grad R and D_R of the new x, computed during the all-reduce
    if (dist) off = align_up(off + sizeof(float) * g->G.nvox);
    L.curvr = off;
    if (dist) off = align_up(off + sizeof(float) * g->G.nvox);
    L.flag = off;
    off = align_up(off + sizeof(int));
    L.dsum = off;
    off = align_up(off + sizeof(double));
    L.total = off;
    return L;
}

static ct_status validate_params(const ct_geom* g, const oslalm_params* p) {
    if (!p) return fail(CT_E_CONFIG, "oslalm_params is NULL");
    if (p->M < 1 || p->M > g->d.na) return fail(CT_E_CONFIG, "M = %d outside [1, na = %d]", p->M, g->d.na);
    if (!(p->alpha >= 1.0 && p->alpha < 2.0)) return fail(CT_E_CONFIG, "alpha = %g outside [1, 2) (P:334)", p->alpha);
    if (p->rho_mode != OSLALM_RHO_CONTINUATION && p->rho_mode != OSLALM_RHO_FIXED)
        return fail(CT_E_CONFIG, "bad rho_mode");
    if (p->rho_mode == OSLALM_RHO_FIXED && !(p->rho_fixed > 0)) return fail(CT_E_CONFIG, "rho_fixed must be > 0");
    if (p->init_grad != OSLALM_INIT_LAST_SUBSET && p->init_grad != OSLALM_INIT_FULL)
        return fail(CT_E_CONFIG, "bad init_grad");
    if (!(p->box_lo <= p->box_hi)) return fail(CT_E_CONFIG, "box_lo > box_hi");
    if (p->variant != OSLALM_PROPOSED && p->variant != OSLALM_SIMPLE) return fail(CT_E_CONFIG, "bad variant");
    return CT_OK;
}

extern "C" ct_status oslalm_workspace_size(const ct_geom* g, const oslalm_params* p, const ct_dist* dist,
                                           size_t* bytes) {
    if (!g || !bytes) return fail(CT_E_CONFIG, "oslalm_workspace_size: NULL argument");
    ct_status st = validate_params(g, p);
    if (st != CT_OK) return st;
    *bytes = ws_layout(g, p, dist).total;
    return CT_OK;
}

extern "C" double oslalm_rho(int64_t k, double alpha) {
    if (k == 0) return 1.0;
    const double pi = 3.14159265358979323846;
    const double a = pi / (alpha * (double)(k + 1));
    return a * std::sqrt(1.0 - 0.25 * a * a);
}

// one sub-iteration (lines 4-9 of Alg. 1) on stream s; single GPU.
static void enqueue_subiter(const ct_geom* g, const RegParams& rp, Ctl* ctl, float* xa, float* xb, float* xt,
                            const float* y, const float* w, const float* dl, float* gb, float* ht,
                            const float* kappa, float* r, int max_count, float M, float lo, float hi,
                            const SegSched* segs, float* part, cudaStream_t s) {
    launch_update(g->G, rp, ctl, xa, xb, dl, gb, ht, kappa, lo, hi, xt, s);
    if (xt) fwd_pfx(g, ctl, Views{0, 1, 0}, segs, max_count, xt, y, w, r, FWD_RESID, part, s);
    else launch_fwd(g->G, g->vtab, ctl, Views{0, 1, 0}, max_count, xa, xb, y, w, r, FWD_RESID, s);
    launch_back(g->G, g->vtab, ctl, Views{0, 1, 0}, r, M, BK_UPDATE, false, nullptr, gb, ht, s);   // + k advance
}

static ct_status solve_impl(const ct_geom* g, const float* y, const float* w, const ct_reg_desc* r,
                            const float* kappa, const float* d_l, const oslalm_params* p, oslalm_state* st,
                            int n_subiters, const float* x_ref, double* rms_per_iter, const ct_dist* dist,
                            void* workspace, size_t workspace_bytes, ct_stream stream, double* kernel_ms) {
    if (!g || !y || !d_l || !st || !workspace) return fail(CT_E_CONFIG, "oslalm_relaxed_solve: NULL argument");
    if (!st->x || !st->g || !st->htilde) return fail(CT_E_CONFIG, "oslalm_state has NULL arrays");
    if (st->k < 0) return fail(CT_E_CONFIG, "state k < 0");
    if (n_subiters < 0) return fail(CT_E_CONFIG, "n_subiters < 0");
    ct_status stt = validate_params(g, p);
    if (stt != CT_OK) return stt;
    RegParams rp;
    stt = make_reg(g, r, rp);
    if (stt != CT_OK) return stt;
    const WsLayout L = ws_layout(g, p, dist);
    if (workspace_bytes < L.total)
        return fail(CT_E_NOMEM, "workspace %zu < %zu bytes (oslalm_workspace_size)", workspace_bytes, L.total);
    if (dist && dist->device != g->device) return fail(CT_E_CONFIG, "ct_dist device != ct_geom device");

    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    Ctl* ctl = (Ctl*)(ws + L.ctl);
    float* xalt = (float*)(ws + L.xalt);
    float* xt = g->G.dim == 3 ? (float*)(ws + L.xt) : nullptr;
    float* rbuf = (float*)(ws + L.r);
    float* part = (float*)(ws + L.part);   // segmented forward (fwd_nseg_of)
    float* zeta = dist ? (float*)(ws + L.zeta) : nullptr;
    const int nl = local_ranks(dist);
    const long long zstride = (long long)(L.zeta_stride / sizeof(float)), rstride = (long long)(L.r_stride / sizeof(float));
    if (dist && g->G.dim == 3 && dist->world > g->G.nz)
        return fail(CT_E_CONFIG, "%d ranks for %d planes (each rank owns a z-slab)", dist->world, g->G.nz);
    float* gradr = dist ? (float*)(ws + L.gradr) : nullptr;
    float* curvr = dist ? (float*)(ws + L.curvr) : nullptr;
    int* dflag = (int*)(ws + L.flag);
    double* dsum = (double*)(ws + L.dsum);
    const int rank = dist ? dist->rank : 0, world = dist ? dist->world : 1;
    const int M = p->M;
    const int vm_max = (g->d.na + M - 1) / M;
    const int max_count = (vm_max + world - 1) / world;
    if ((long long)max_count * g->G.nt * g->G.ns >= (1LL << 31))
        return fail(CT_E_SHAPE, "subset projection block exceeds 2^31 elements (increase M)");
    const float lo = (float)p->box_lo, hi = std::isinf(p->box_hi) ? 3.0e38f : (float)p->box_hi;
    const int sstride = world * M;   // view stride of a rank's subset (the segmented forward's schedule)
    const SegSched* segs = nullptr;   // the segmented forward's schedule (nullptr: unsegmented)
    const int nseg = xt ? fwd_nseg_of(g, max_count) : 0;
    if (nseg) {
        ct_status e = seg_sched(g, sstride, max_count, nseg, &segs);
        if (e != CT_OK) return e;
    }

    std::vector<Ctl> hctl(nl);
    for (int q = 0; q < nl; q++) {
        Ctl& h = hctl[q];
        memset(&h, 0, sizeof(h));
        h.k = st->k;
        h.k_base = st->k;
        h.M = M;
        h.na = g->d.na;
        h.rank = dist && dist->local ? q : rank;
        h.world = world;
        h.rho_fixed_mode = p->rho_mode == OSLALM_RHO_FIXED;
        h.simple = p->variant == OSLALM_SIMPLE;
        h.alpha = (float)p->alpha;
        h.rho_fixed = (float)p->rho_fixed;
    }
    // pageable source: the copy is staged before cudaMemcpyAsync returns
    CT_CUDA(cudaMemcpyAsync(ctl, hctl.data(), sizeof(Ctl) * nl, cudaMemcpyHostToDevice, s));

    NvtxRange nv_solve(dist ? (dist->local ? "oslalm_relaxed_solve (local ranks)" : "oslalm_relaxed_solve (NCCL)")
                             : "oslalm_relaxed_solve");
    // ---- line 1: rho = 1, zeta = g = M grad L_M(x), h = D_L x - zeta  (htilde = zeta)
    if (st->k == 0) {
        NvtxRange nv1("Algorithm 1 line 1");
        float* zdst = dist ? zeta : st->g;
        // every local rank's partial gradient is accumulated in rank order into zdst
        bool first = true;
        for (int q = 0; q < nl; q++) {
            const int rk = dist && dist->local ? q : rank;
            if (p->init_grad == OSLALM_INIT_LAST_SUBSET) {
                const int m = M - 1;
                const int vm = (g->d.na - m + M - 1) / M;
                const int cnt = (vm - rk + world - 1) / world;
                Views vv{m + rk * M, world * M, cnt};
                if (cnt > 0) {
                    launch_fwd(g->G, g->vtab, nullptr, vv, cnt, st->x, st->x, y, w, rbuf, FWD_RESID, s);
                    launch_back(g->G, g->vtab, nullptr, vv, rbuf, (float)M, first ? BK_WRITE : BK_ACCUM, false, zdst,
                                nullptr, nullptr, s);
                    first = false;
                }
            } else {
                const int mine = (g->d.na - rk + world - 1) / world;
                for (int c0 = 0; c0 < mine; c0 += max_count) {
                    const int cnt = std::min(max_count, mine - c0);
                    Views vv{rk + c0 * world, world, cnt};
                    launch_fwd(g->G, g->vtab, nullptr, vv, cnt, st->x, st->x, y, w, rbuf, FWD_RESID, s);
                    launch_back(g->G, g->vtab, nullptr, vv, rbuf, 1.0f, first ? BK_WRITE : BK_ACCUM, false, zdst,
                                nullptr, nullptr, s);
                    first = false;
                }
            }
        }
        if (first) CT_CUDA(cudaMemsetAsync(zdst, 0, sizeof(float) * g->G.nvox, s));
        if (dist && !dist->local)
            CT_NCCL(ncclAllReduce(zeta, zeta, (size_t)g->G.nvox, ncclFloat, ncclSum, dist->comm, s));
        launch_init_from_zeta(g->G, zdst, st->g, st->htilde, s);
        stt = check_async();
        if (stt != CT_OK) return stt;
    }

    // ---- sub-iterations
    const float Mf = (float)M;
    int done = 0;
    int iter_out = 0;
    long long kcur = st->k;
    cudaGraphExec_t exec = nullptr;
    const int kernels_per_subiter = segs ? 4 : 3;   // + the segment reduce
    if (!dist && !kernel_ms && n_subiters > 0) {
        GraphKey key;
        key.ptrs = {(uintptr_t)ctl, (uintptr_t)st->x, (uintptr_t)xalt, (uintptr_t)y, (uintptr_t)w,
                    (uintptr_t)d_l, (uintptr_t)st->g, (uintptr_t)st->htilde, (uintptr_t)kappa, (uintptr_t)rbuf,
                    (uintptr_t)xt};
        key.vals = {(double)M, p->alpha, (double)p->rho_mode, p->rho_fixed, (double)lo, (double)hi, (double)p->variant,
                    (double)rp.potential, (double)rp.delta, (double)rp.n_dirs, (double)rp.maxcurv, (double)rp.q,
                    (double)nseg};
        for (int i = 0; i < 13; i++) key.vals.push_back(rp.beta[i]);
        std::lock_guard<std::mutex> lk(const_cast<ct_geom*>(g)->mu);
        auto it = g->graphs.find(key);
        if (it != g->graphs.end()) {
            exec = it->second;
        } else {
            cudaStream_t cs = g->cap_stream;
            CT_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            {
                // the sub-iteration's kernels chained by programmatic dependent launch: each grid
                // is scheduled during its predecessor's tail and waits for it (griddepcontrol)
                PdlScope pdl(CTR_PDL != 0);
                enqueue_subiter(g, rp, ctl, st->x, xalt, xt, y, w, d_l, st->g, st->htilde, kappa, rbuf, max_count,
                                Mf, lo, hi, segs, part, cs);
            }
            cudaGraph_t graph;
            cudaError_t e = cudaStreamEndCapture(cs, &graph);
            if (e != cudaSuccess) return fail(CT_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
            e = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) return fail(CT_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
            launches_add(-kernels_per_subiter);  // capture is not a launch; replays are counted below
            const_cast<ct_geom*>(g)->graphs[key] = exec;
        }
    }
    std::vector<cudaEvent_t> evs;
    if (kernel_ms) {
        evs.resize((size_t)n_subiters * 5);
        for (auto& e : evs) CT_CUDA(cudaEventCreate(&e));
    }
    // multi-GPU: the owner slabs this process updates (all of them in a local emulation) and the
    // collectives of the partial-gradient reduction
    // (2-D: one owner of the whole image on every rank: the update is replicated after the all-reduce)
    const bool split = g->G.dim == 3;
    const int own0 = split && dist && !dist->local ? rank : 0;
    const int own1 = !split ? 1 : dist && !dist->local ? rank + 1 : nl;
    auto reduce_partials = [&](cudaStream_t cs) -> ct_status {
        const DGeom& G = g->G;
        if (dist->local) {
            if (nl > 1) launch_sum_partials(zeta, nl, zstride, G.nvox, cs);
            return check_async();
        }
        if (G.dim != 3 || world == 1) {
            CT_NCCL(ncclAllReduce(zeta, zeta, (size_t)G.nvox, ncclFloat, ncclSum, dist->comm, cs));
        } else if (G.nz % world == 0) {
            const size_t cnt = (size_t)(G.nz / world) * G.nxy;
            CT_NCCL(ncclReduceScatter(zeta, zeta + (size_t)rank * cnt, cnt, ncclFloat, ncclSum, dist->comm, cs));
        } else {
            CT_NCCL(ncclGroupStart());
            for (int q = 0; q < world; q++) {
                int a, nzq;
                owner_slab(G, q, world, &a, &nzq);
                float* b = zeta + (size_t)a * G.nxy;
                CT_NCCL(ncclReduce(b, b, (size_t)nzq * G.nxy, ncclFloat, ncclSum, q, dist->comm, cs));
            }
            CT_NCCL(ncclGroupEnd());
        }
        return CT_OK;
    };
    auto all_gather = [&](float* buf, cudaStream_t cs) -> ct_status {
        const DGeom& G = g->G;
        if (dist->local || G.dim != 3 || world == 1) return CT_OK;   // every slab already in place
        if (G.nz % world == 0) {
            const size_t cnt = (size_t)(G.nz / world) * G.nxy;
            CT_NCCL(ncclAllGather(buf + (size_t)rank * cnt, buf, cnt, ncclFloat, dist->comm, cs));
        } else {
            CT_NCCL(ncclGroupStart());
            for (int q = 0; q < world; q++) {
                int a, nzq;
                owner_slab(G, q, world, &a, &nzq);
                float* b = buf + (size_t)a * G.nxy;
                CT_NCCL(ncclBroadcast(b, b, (size_t)nzq * G.nxy, ncclFloat, q, dist->comm, cs));
            }
            CT_NCCL(ncclGroupEnd());
        }
        return CT_OK;
    };
    bool pending = false;  // multi-GPU: zeta of the previous sub-iteration not yet folded into g, htilde
    while (done < n_subiters) {
        cudaEvent_t* ev = kernel_ms ? &evs[(size_t)done * 5] : nullptr;
        if (exec) {
            CT_CUDA(cudaGraphLaunch(exec, s));
            launches_add(kernels_per_subiter);
        } else if (!dist) {
            if (ev) CT_CUDA(cudaEventRecord(ev[0], s));
            launch_update(g->G, rp, ctl, st->x, xalt, d_l, st->g, st->htilde, kappa, lo, hi, xt, s);
            if (ev) CT_CUDA(cudaEventRecord(ev[1], s));
            if (xt) fwd_pfx(g, ctl, Views{0, 1, 0}, segs, max_count, xt, y, w, rbuf, FWD_RESID, part, s);
            else launch_fwd(g->G, g->vtab, ctl, Views{0, 1, 0}, max_count, st->x, xalt, y, w, rbuf, FWD_RESID, s);
            if (ev) CT_CUDA(cudaEventRecord(ev[2], s));
            launch_back(g->G, g->vtab, ctl, Views{0, 1, 0}, rbuf, Mf, BK_UPDATE, false, nullptr, st->g, st->htilde, s);
            if (ev) CT_CUDA(cudaEventRecord(ev[3], s));   // (the back-projection's last block advanced k)
            if (ev) CT_CUDA(cudaEventRecord(ev[4], s));
        } else {
            // Multi-GPU sub-iteration: this rank's views are projected, the partial
            // back-projections are reduce-scattered by z-slab (3-D; all-reduced in 2-D), the owner of
            // each slab folds zeta into g, htilde and updates x on its slab only (the stencil of that
            // slab ran on the side stream while the projections and the reduction were in flight),
            // x+ is all-gathered and its z-prefix rebuilt for the next forward.  A local emulation
            // (ct_dist_create_local) runs every rank's projections in turn into its own partial
            // buffer, sums them in rank order and updates every slab: the same data flow on one GPU.
            const DGeom& G = g->G;
            float* xin = (done & 1) ? xalt : st->x;
            float* xout = (done & 1) ? st->x : xalt;
            const bool last = done + 1 == n_subiters;
            if (ev) CT_CUDA(cudaEventRecord(ev[0], s));
            if (pending) CT_CUDA(cudaStreamWaitEvent(s, dist->ev_sten, 0));
            for (int q = own0; q < own1; q++) {
                int a, nzq;
                owner_slab(G, q, world, &a, &nzq);
                if (nzq == 0) continue;
                const size_t off = (size_t)a * G.nxy;
                const DGeom S = sub_geom(G, a, nzq);
                const bool hl = a > 0, hh = a + nzq < G.nz;
                if (!pending)
                    launch_update_halo(S, rp, ctl, st->x + off, xalt + off, d_l + off, st->g + off, st->htilde + off,
                                       lo, hi, nullptr, hl, hh, s, kappa ? kappa + off : nullptr);
                else
                    launch_update_pre(S, ctl, xin + off, xout + off, d_l + off, st->g + off, st->htilde + off,
                                      zeta + off, gradr + off, curvr + off, lo, hi, nullptr, s);
            }
            if (pending) launch_advance(ctl, s, nl);
            stt = all_gather(xout, s);
            if (stt != CT_OK) return stt;
            if (xt) launch_zprefix(G, xout, xt, s);
            if (ev) CT_CUDA(cudaEventRecord(ev[1], s));
            if (!last) {
                // the stencil of x+ feeds the next sub-iteration of this call only: the last
                // sub-iteration's fold (below) completes the state without it
                CT_CUDA(cudaEventRecord(dist->ev_x, s));
                CT_CUDA(cudaStreamWaitEvent(dist->side, dist->ev_x, 0));
                for (int q = own0; q < own1; q++) {
                    int a, nzq;
                    owner_slab(G, q, world, &a, &nzq);
                    if (nzq == 0) continue;
                    const size_t off = (size_t)a * G.nxy;
                    launch_reg(sub_geom(G, a, nzq), rp, xout + off, kappa ? kappa + off : nullptr, gradr + off,
                               curvr + off, dist->side, a > 0, a + nzq < G.nz);
                }
                CT_CUDA(cudaEventRecord(dist->ev_sten, dist->side));
            }
            for (int q = 0; q < nl; q++) {
                float* rq = rbuf + q * rstride;
                if (xt) fwd_pfx(g, ctl + q, Views{0, 1, 0}, segs, max_count, xt, y, w, rq, FWD_RESID, part, s);
                else launch_fwd(G, g->vtab, ctl + q, Views{0, 1, 0}, max_count, st->x, xalt, y, w, rq, FWD_RESID, s);
            }
            if (ev) CT_CUDA(cudaEventRecord(ev[2], s));
            for (int q = 0; q < nl; q++)
                launch_back(G, g->vtab, ctl + q, Views{0, 1, 0}, rbuf + q * rstride, Mf, BK_WRITE, false,
                            zeta + q * zstride, nullptr, nullptr, s);
            if (ev) CT_CUDA(cudaEventRecord(ev[3], s));
            stt = reduce_partials(s);
            if (stt != CT_OK) return stt;
            pending = true;
            if (last) {
                // fold the last zeta (lines 7-8) on the owned slabs, advance, and replicate g, htilde:
                // the state is complete (and identical on every rank) on return
                for (int q = own0; q < own1; q++) {
                    int a, nzq;
                    owner_slab(G, q, world, &a, &nzq);
                    if (nzq == 0) continue;
                    const size_t off = (size_t)a * G.nxy;
                    launch_gh_update(sub_geom(G, a, nzq), ctl, zeta + off, st->g + off, st->htilde + off, s);
                }
                launch_advance(ctl, s, nl);
                stt = all_gather(st->g, s);
                if (stt == CT_OK) stt = all_gather(st->htilde, s);
                if (stt != CT_OK) return stt;
                pending = false;
            }
            if (ev) CT_CUDA(cudaEventRecord(ev[4], s));
        }
        done++;
        kcur++;
        if (x_ref && rms_per_iter && kcur % M == 0) {
            const float* xc = (done & 1) ? xalt : st->x;
            CT_CUDA(cudaMemsetAsync(dsum, 0, sizeof(double), s));
            launch_check(g->G, xc, x_ref, dflag, dsum, s);
            double hs = 0.0;
            CT_CUDA(cudaMemcpyAsync(&hs, dsum, sizeof(double), cudaMemcpyDeviceToHost, s));
            CT_CUDA(cudaStreamSynchronize(s));
            rms_per_iter[iter_out++] = std::sqrt(hs / (double)g->G.nvox);
        }
    }
    if (kernel_ms) {
        CT_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; q < 4; q++) kernel_ms[q] = 0.0;
        for (int it = 0; it < n_subiters; it++) {
            for (int q = 0; q < 4; q++) {
                float ms = 0.f;
                CT_CUDA(cudaEventElapsedTime(&ms, evs[(size_t)it * 5 + q], evs[(size_t)it * 5 + q + 1]));
                kernel_ms[q] += ms;
            }
        }
        for (auto& e : evs) cudaEventDestroy(e);
    }
    if (n_subiters & 1) CT_CUDA(cudaMemcpyAsync(st->x, xalt, sizeof(float) * g->G.nvox, cudaMemcpyDeviceToDevice, s));
    st->k += n_subiters;
    // finiteness of the returned image (K7)
    CT_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), s));
    launch_check(g->G, st->x, nullptr, dflag, nullptr, s);
    int hflag = 0;
    CT_CUDA(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    stt = check_async();
    if (stt != CT_OK) return stt;
    if (hflag) return fail(CT_E_NUMERIC, "non-finite values in x after sub-iteration %lld", (long long)st->k);
    return CT_OK;
}

extern "C" ct_status oslalm_relaxed_solve(const ct_geom* g, const float* y, const float* w, const ct_reg_desc* r,
                                          const float* kappa, const float* d_l, const oslalm_params* p,
                                          oslalm_state* st, int n_subiters, const float* x_ref,
                                          double* rms_per_iter, const ct_dist* dist, void* workspace,
                                          size_t workspace_bytes, ct_stream stream) {
    return solve_impl(g, y, w, r, kappa, d_l, p, st, n_subiters, x_ref, rms_per_iter, dist, workspace,
                      workspace_bytes, stream, nullptr);
}

extern "C" ct_status oslalm_profile(const ct_geom* g, const float* y, const float* w, const ct_reg_desc* r,
                                    const float* kappa, const float* d_l, const oslalm_params* p, oslalm_state* st,
                                    int n_subiters, const ct_dist* dist, void* workspace, size_t workspace_bytes,
                                    ct_stream stream, double* kernel_ms) {
    if (!kernel_ms) return fail(CT_E_CONFIG, "oslalm_profile: kernel_ms is NULL");
    return solve_impl(g, y, w, r, kappa, d_l, p, st, n_subiters, nullptr, nullptr, dist, workspace,
                      workspace_bytes, stream, kernel_ms);
}

extern "C" ct_status oslalm_residual(const ct_geom* g, const oslalm_params* p, const ct_dist* dist, int64_t k,
                                     const void* workspace, size_t workspace_bytes, float* r_out, ct_stream stream) {
    if (!g || !workspace || !r_out) return fail(CT_E_CONFIG, "oslalm_residual: NULL argument");
    ct_status st = validate_params(g, p);
    if (st != CT_OK) return st;
    if (k < 1) return fail(CT_E_CONFIG, "oslalm_residual: k = %lld, no sub-iteration done", (long long)k);
    const WsLayout L = ws_layout(g, p, dist);
    if (workspace_bytes < L.total) return fail(CT_E_NOMEM, "workspace %zu < %zu bytes", workspace_bytes, L.total);
    const int rank = dist ? dist->rank : 0, world = dist ? dist->world : 1;
    const int M = p->M, m = (int)((k - 1) % M);
    const int vm = (g->d.na - m + M - 1) / M;
    const int cnt = std::max(0, (vm - rank + world - 1) / world);
    if (cnt == 0) return CT_OK;
    DeviceGuard guard(g->device);
    const float* rbuf = (const float*)((const char*)workspace + L.r);
    launch_unfold_lz(g->G, cnt, rbuf, r_out, (cudaStream_t)stream);
    return check_async();
}

extern "C" ct_status ct_count_nnz(const ct_geom* g, ct_views v, uint64_t* d_count, ct_stream s) {
    if (!g || !d_count) return fail(CT_E_CONFIG, "ct_count_nnz: NULL argument");
    ct_status st = check_views(g, v);
    if (st != CT_OK) return st;
    DeviceGuard guard(g->device);
    launch_count(g->G, g->vtab, to_views(v), (unsigned long long*)d_count, (cudaStream_t)s);
    return check_async();
}

extern "C" ct_status ct_count_work(const ct_geom* g, ct_views v, uint64_t* d_counts, ct_stream s) {
    if (!g || !d_counts) return fail(CT_E_CONFIG, "ct_count_work: NULL argument");
    ct_status st = check_views(g, v);
    if (st != CT_OK) return st;
    DeviceGuard guard(g->device);
    launch_count_work(g->G, g->vtab, to_views(v), (unsigned long long*)d_counts, (cudaStream_t)s);
    return check_async();
}

extern "C" ct_status oslalm_state_h(const ct_geom* g, const float* d_l, const oslalm_state* st, float* h_out,
                                    ct_stream s) {
    if (!g || !d_l || !st || !st->x || !st->htilde || !h_out) return fail(CT_E_CONFIG, "oslalm_state_h: NULL argument");
    DeviceGuard guard(g->device);
    launch_state_h(g->G, d_l, st->x, st->htilde, h_out, (cudaStream_t)s);
    return check_async();
}

extern "C" ct_status ct_sino_upload(const ct_geom* g, const float* host, ct_views v, float* dev, ct_stream s) {
    if (!g || !host || !dev) return fail(CT_E_CONFIG, "ct_sino_upload: NULL argument");
    ct_status st = check_views(g, v);
    if (st != CT_OK) return st;
    if (v.count == 0) return CT_OK;
    DeviceGuard guard(g->device);
    const size_t row = (size_t)g->d.nt * (size_t)g->d.ns;   // floats per view
    const size_t off = (size_t)v.start * row, pitch = (size_t)v.stride * row * sizeof(float);
    CT_CUDA(cudaMemcpy2DAsync(dev + off, pitch, host + off, pitch, row * sizeof(float), (size_t)v.count,
                              cudaMemcpyHostToDevice, (cudaStream_t)s));
    return CT_OK;
}

extern "C" ct_status ct_sync(ct_stream s) {
    CT_CUDA(cudaStreamSynchronize((cudaStream_t)s));
    return check_async();
}

// ------------------------------------------------------------------ NCCL
// ------------------------------------------------------------------ accessors for zslab.cu
ct_status ctr_fail(ct_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}
const DGeom& ctr_geom_dev(const ct_geom* g) { return g->G; }
const float4* ctr_geom_vtab(const ct_geom* g) { return g->vtab; }
const ct_geom_desc& ctr_geom_desc(const ct_geom* g) { return g->d; }
int ctr_geom_device(const ct_geom* g) { return g->device; }
ncclComm_t ctr_dist_comm(const ct_dist* d) { return d->comm; }
int ctr_dist_rank(const ct_dist* d) { return d->rank; }
int ctr_dist_world(const ct_dist* d) { return d->world; }
ct_status ctr_make_reg(const ct_geom* g, const ct_reg_desc* r, RegParams& rp) { return make_reg(g, r, rp); }
ct_status ctr_validate_params(const ct_geom* g, const oslalm_params* p) { return validate_params(g, p); }

extern "C" ct_status ct_nccl_unique_id(unsigned char id[128]) {
    if (!id) return fail(CT_E_CONFIG, "id is NULL");
    ncclUniqueId u;
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId size");
    CT_NCCL(ncclGetUniqueId(&u));
    memcpy(id, u.internal, 128);
    return CT_OK;
}

extern "C" ct_status ct_dist_create(int rank, int world, const unsigned char id[128], int device, ct_dist** out) {
    if (!out || !id) return fail(CT_E_CONFIG, "ct_dist_create: NULL argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(CT_E_CONFIG, "bad rank %d / world %d", rank, world);
    DeviceGuard guard(device);
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclComm_t comm;
    CT_NCCL(ncclCommInitRank(&comm, world, u, rank));
    ct_dist* d = new ct_dist{comm, rank, world, device, nullptr, nullptr, nullptr, false};
    int lo = 0, hi = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&d->side, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_x, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_sten, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        ct_dist_destroy(d);
        return fail(CT_E_CUDA, "ct_dist_create: %s", cudaGetErrorString(e));
    }
    *out = d;
    return CT_OK;
}

extern "C" ct_status ct_dist_create_local(int world, int device, ct_dist** out) {
    if (!out) return fail(CT_E_CONFIG, "ct_dist_create_local: NULL argument");
    *out = nullptr;
    if (world < 1 || world > 64) return fail(CT_E_CONFIG, "local world %d outside [1, 64]", world);
    int ndev = 0;
    CT_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CT_E_CONFIG, "device %d not present", device);
    DeviceGuard guard(device);
    ct_dist* d = new ct_dist{nullptr, 0, world, device, nullptr, nullptr, nullptr, true};
    int lo = 0, hi = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&d->side, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_x, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_sten, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        ct_dist_destroy(d);
        return fail(CT_E_CUDA, "ct_dist_create_local: %s", cudaGetErrorString(e));
    }
    *out = d;
    return CT_OK;
}

extern "C" void ct_dist_destroy(ct_dist* d) {
    if (!d) return;
    DeviceGuard guard(d->device);
    if (d->ev_sten) cudaEventDestroy(d->ev_sten);
    if (d->ev_x) cudaEventDestroy(d->ev_x);
    if (d->side) cudaStreamDestroy(d->side);
    if (d->comm) ncclCommDestroy(d->comm);
    delete d;
}

extern "C" int64_t ct_launch_count(void) { return g_launches.load(); }

extern "C" const char* ct_last_error(void) { return g_err.c_str(); }
