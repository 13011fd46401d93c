/*
 * ctrecon.h — C-ABI of the B200-native relaxed OS-LALM hot path
 * (Nien & Fessler, "Relaxed Linearized Algorithms for Faster X-Ray CT Image
 * Reconstruction", arXiv 1512.04564; the text is PAPER.md, cited as P:line).
 *
 * Library: paper_1512_04564_b200/libctrecon.so (sm_100a).  Every function is
 * extern "C", returns ct_status (or void), never throws, and validates all
 * arguments BEFORE launching anything: a call that returns an error has no
 * side effects.  ct_last_error() gives a thread-local message.
 *
 * Memory: every float* / int64_t* array argument is a DEVICE pointer owned by
 * the caller unless stated otherwise.  The library allocates device memory
 * only for the small per-view table inside ct_geom and for the NCCL
 * communicator inside ct_dist; the solver's scratch is a caller-provided
 * workspace sized by oslalm_workspace_size().  All work is asynchronous on
 * the given stream; asynchronous CUDA faults surface as CT_E_CUDA from the
 * next call or from ct_sync().
 *
 * Layouts (C order, last index fastest):
 *   volume      float[nz][ny][nx]          (2-D: nz = 1)
 *   projections float[views][nt][ns]       (2-D: nt = 1), view index first
 *   full sinogram arrays (y, w) hold all na views; a view descriptor selects
 *   rows of them.
 */
#ifndef CTRECON_H
#define CTRECON_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ct_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    CT_OK = 0,
    CT_E_SHAPE = 1,    /* inconsistent sizes / view index out of range          */
    CT_E_CONFIG = 2,   /* bad parameter: alpha, rho, M, delta, box, geometry      */
    CT_E_NUMERIC = 3,  /* non-finite iterate detected                             */
    CT_E_DIVERGED = 4, /* reserved (cost guard)                                   */
    CT_E_CUDA = 5,     /* CUDA runtime / launch fault                             */
    CT_E_NCCL = 6,     /* NCCL fault                                              */
    CT_E_NOMEM = 7     /* workspace too small                                     */
} ct_status;

typedef enum { CT_DET_FLAT = 0, CT_DET_ARC = 1 } ct_det_shape;

/*
 * Scanner geometry ("A is the forward projection matrix of a CT
 * scan"; the paper cites a separable-footprint projector [long:10:3fa] and
 * does not define it — the projector implemented here is DESIGN.md §3 /
 * SURVEY.md 8c.1).  Lengths in mm, angles in degrees.
 *   voxel centre i:  (i - (nx-1)/2) dx + offset_x  (likewise y, z)
 *   view v:          beta_v = orbit_start + orbit * v / na
 *                    source (Dso cos beta, Dso sin beta, z_s(v)),
 *                    z_s(v) = source_z0 + v * pitch * nt*dt*Dso/Dsd * (orbit/360) / na
 *   column centre s: (s - (ns-1)/2 - offset_s) * Delta, Delta = ds (flat, mm at
 *                    the detector) or ds/Dsd (arc, radians)
 *   row centre t:    (t - (nt-1)/2 - offset_t) * dt
 * dim = 2: fan beam, nz = nt = 1, z ignored.  dim = 3: cone beam (pitch 0 =
 * axial, > 0 = helical).
 */
typedef struct {
    int32_t dim;
    int32_t nx, ny, nz;
    double dx, dy, dz;
    double offset_x, offset_y, offset_z;
    int32_t det_shape; /* ct_det_shape */
    int32_t ns, nt;
    double ds, dt;
    double offset_s, offset_t;
    double dso, dsd;
    int32_t na;
    double orbit_deg, orbit_start_deg, pitch, source_z0;
} ct_geom_desc;

/* Arithmetic progression of views {start, start+stride, ...} (count terms).
 * Subset m of M ("L_m ... the m-th subset"; reading R4):
 * {m, M, ceil((na-m)/M)}.  Every index must be < na (else CT_E_SHAPE). */
typedef struct {
    int32_t start, stride, count;
} ct_views;

/* Edge-preserving regulariser of Eq. 35:
 *   R(x) = sum_i beta_i sum_n kappa_n kappa_{n+s_i} phi([C_i x]_n)
 * over n_dirs directions (13 in 3-D = 26 neighbours; 4 in 2-D).  The
 * direction order is fixed (offsets in voxels):
 *   0 (1,0,0) 1 (0,1,0) 2 (1,1,0) 3 (1,-1,0) 4 (0,0,1) 5 (1,0,1) 6 (-1,0,1)
 *   7 (0,1,1) 8 (0,-1,1) 9 (1,1,1) 10 (-1,1,1) 11 (1,-1,1) 12 (-1,-1,1)
 * Potentials: quadratic t^2/2; hyperbola delta^2(sqrt(1+(t/delta)^2)-1);
 * Fair delta^2(|t/delta| - log(1+|t/delta|)); q-GGMRF with p = 2,
 * (t^2/2)/(1 + |t/delta|^(2-q)), 1 <= q <= 2 (Thibault et al. 2007, the
 * chest experiment's regulariser).  delta > 0.
 * Curvature D_R: CT_CURV_HUBER = 2 sum beta kappa kappa
 * omega(x_j - x_n), omega = phi'(t)/t (Huber's curvature, the paper's
 * choice); CT_CURV_MAX = 2 sum beta kappa kappa omega(0), the maximum
 * curvature (the constant majorizer the paper's theorems assume). */
typedef enum { CT_POT_QUADRATIC = 0, CT_POT_HYPERBOLA = 1, CT_POT_FAIR = 2, CT_POT_QGGMRF = 3 } ct_potential;
typedef enum { CT_CURV_HUBER = 0, CT_CURV_MAX = 1 } ct_curvature;

typedef struct {
    int32_t potential; /* ct_potential */
    double delta;
    int32_t n_dirs;    /* 4 or 13 */
    double beta[13];   /* beta_i >= 0 */
    int32_t curvature; /* ct_curvature */
    double q;          /* q-GGMRF exponent, 1 <= q <= 2 (ignored by the other potentials) */
} ct_reg_desc;

typedef enum { OSLALM_RHO_CONTINUATION = 0, OSLALM_RHO_FIXED = 1 } oslalm_rho_mode;
typedef enum { OSLALM_INIT_LAST_SUBSET = 0, OSLALM_INIT_FULL = 1 } oslalm_init_grad;

/* Which OS-LALM recursion:
 *   OSLALM_PROPOSED  Algorithm 1, s = rho (D_L x - h) + (1 - rho) g
 *   OSLALM_SIMPLE    Algorithm 2, s = rho zeta + (1 - rho) g, no h
 * alpha = 1 reverts either to the unrelaxed OS-LALM; SIMPLE with
 * rho_mode FIXED, rho_fixed = 1 is OS-SQS [erdogan:99:osa] (s = zeta, step
 * (D_L + D_R)^{-1}), the paper's conventional baseline. */
typedef enum { OSLALM_PROPOSED = 0, OSLALM_SIMPLE = 1 } oslalm_variant;

/* Algorithm 1 inputs ("M >= 1, 1 <= alpha < 2").  box = [box_lo, box_hi]
 * is Omega; box_hi = +inf for the non-negativity constraint. */
typedef struct {
    int32_t M;
    double alpha;
    int32_t rho_mode;  /* oslalm_rho_mode; CONTINUATION = Eq. 37 */
    double rho_fixed;  /* used when rho_mode == FIXED, > 0 */
    int32_t init_grad; /* oslalm_init_grad; LAST_SUBSET = P:336 literally */
    double box_lo, box_hi;
    int32_t variant;   /* oslalm_variant; 0 = Algorithm 1 */
} oslalm_params;

/*
 * Solver state (device arrays of the volume size, caller-owned):
 *   x       image ("x"), in/out
 *   g       P:336-342 "g" (= A'(u - y))
 *   htilde  D_L x - h, where h is Algorithm 1's h.  The library
 *           carries htilde instead of h: the two are algebraically identical
 *           updates, but htilde avoids the float32
 *           cancellation of D_L x - h in line 4.  oslalm_state_h() recovers h.
 *           With variant OSLALM_SIMPLE this array holds zeta, the last
 *           subset gradient (Algorithm 2 has no h).
 *   k       number of sub-iterations done (Eq. 37 counter).  k == 0
 *           on entry runs line 1 of Alg. 1 (rho = 1, zeta = g = M grad L_M(x),
 *           h = D_L x - zeta) before the first sub-iteration.
 */
typedef struct {
    float* x;
    float* g;
    float* htilde;
    int64_t k;
} oslalm_state;

typedef struct ct_geom ct_geom; /* opaque; immutable after creation */
typedef struct ct_dist ct_dist; /* opaque NCCL communicator wrapper  */

/* Geometry handle on CUDA device `device`.  Precomputes the per-view table
 * (cos beta, sin beta, z_s) in double, stored as float on the device.
 * Errors: CT_E_CONFIG (non-positive sizes/spacings, dso <= 0, dsd <= 0,
 * source inside the volume's circumscribed cylinder, footprint wider than
 * 16 detector columns), CT_E_CUDA. */
ct_status ct_geom_create(const ct_geom_desc* d, int device, ct_geom** out);
void ct_geom_destroy(ct_geom* g);

/* p = A x on views v (Eq. 36 is NOT applied: no weights).
 * x: volume; proj: float[v.count][nt][ns] (overwritten). */
ct_status ct_forward(const ct_geom* g, const float* x, ct_views v, float* proj, ct_stream s);

/* p = A x on views v through the z-prefix path of the solver's forward
 * projection (Algorithm 1 line 6): the cumulative sums
 * of x along z are formed first (float2 (A_k, x_k) per voxel, z fastest,
 * in the workspace) and each detector row's F2-weighted sum is one difference
 * of the interpolated cumulative.  Same entries as ct_forward up to float32
 * rounding; this is the kernel oslalm_relaxed_solve runs (with the residual
 * epilogue instead of the plain one).  2-D geometries: same as ct_forward.
 * workspace: device, 16-byte aligned, >= ct_zprefix_size bytes (contents
 * overwritten).  Errors: CT_E_CONFIG (NULL, alignment), CT_E_SHAPE (views),
 * CT_E_NOMEM (workspace), CT_E_CUDA. */
ct_status ct_zprefix_size(const ct_geom* g, size_t* bytes);
ct_status ct_forward_zprefix(const ct_geom* g, const float* x, ct_views v, float* proj, void* workspace,
                             size_t workspace_bytes, ct_stream s);

/* Segmented z-prefix forward (the same A x as above):
 * the wedge of every detector-column block is walked in nseg slab segments,
 * scheduled so that resident blocks share one xy tile of the z-prefix in L2,
 * and the segments' raw row sums are added in segment order (deterministic)
 * before the epilogue.
 * nseg: -1 automatic (the default): 16 when the z-prefix array exceeds 512 MB
 * (c5, where every view otherwise re-streams its band of it from HBM); for
 * 3-D volumes of at least 256 x 256 columns as many (<= 8) as keep the
 * partial sums of one launch within 96 MB (c4: 3, c3: 8); else off.  0 or 1:
 * off; 2..64: forced.  Applies to ct_forward_zprefix (launches of <= 128
 * views) and oslalm_relaxed_solve / oslalm_profile (one subset per launch) of
 * this geometry; it changes ct_zprefix_size and oslalm_workspace_size (query
 * them after setting it).  Frees the geometry's cached solve graphs; call it
 * while no work of this geometry is in flight.  ct_geom_fwd_segments returns
 * the count used for a launch of `views` views (0 = unsegmented).
 * Errors: CT_E_CONFIG (NULL, nseg outside [-1, 64]). */
ct_status ct_geom_set_fwd_segments(ct_geom* g, int nseg);
ct_status ct_geom_fwd_segments(const ct_geom* g, int views, int* nseg);

/* x_out (=|+=) scale * A' proj on views v.
 * proj: float[v.count][nt][ns]; accumulate != 0 adds into x_out. */
ct_status ct_back(const ct_geom* g, const float* proj, ct_views v, float scale, int accumulate, float* x_out,
                  ct_stream s);

/* SQS diagonal D_L = diag(A' W A 1) over all na views.
 * w: full sinogram weights float[na][nt][ns] (NULL = all ones); d_out: volume.
 * workspace: device scratch of >= nt*ns*4 bytes (more = fewer chunks).
 * dist != NULL: each rank projects its share of views and the result is
 * summed with ncclAllReduce (identical on all ranks). */
ct_status ct_sqs_diag(const ct_geom* g, const float* w, const ct_dist* dist, float* d_out, void* workspace,
                      size_t workspace_bytes, ct_stream s);

/* Initial image by filtered back-projection ("an initial (FBP)
 * image"; the paper does not define it): textbook fan-beam FBP (equiangular
 * arc / equispaced flat detector; Kak & Slaney ch. 3.4) for 2-D, Feldkamp
 * (FDK) for axial cone scans; Ram-Lak filter, bilinear interpolation,
 * full 360-degree orbit (oracle/fbp.py).
 * proj: line integrals float[na][nt][ns] (all views); x_out: volume.
 * workspace >= na*nt*ns*4 bytes (the filtered sinogram).
 * Errors: CT_E_CONFIG (helical scan, orbit != 360 degrees, NULL,
 * ns > 18000), CT_E_NOMEM, CT_E_CUDA. */
ct_status ct_fbp(const ct_geom* g, const float* proj, float* x_out, void* workspace, size_t workspace_bytes,
                 ct_stream s);

/* Resolution-uniformity weights of the regulariser (kappa_n, cited
 * to [fessler:96:srp]; the formula is SPEC.md:529-531's reading):
 *   kappa_j = sqrt([A'W1]_j / [A'1]_j),  0/0 = 1,
 * over all views, A' the exact transpose of ct_forward (L_z included).
 * w: full sinogram weights float[na][nt][ns] (NULL = all ones -> kappa = 1).
 * kappa_out: volume.  workspace: >= (nvox + nt*ns) * 4 bytes (more = fewer
 * chunks).  Errors: CT_E_CONFIG (NULL), CT_E_NOMEM, CT_E_CUDA. */
ct_status ct_kappa_weights(const ct_geom* g, const float* w, float* kappa_out, void* workspace,
                           size_t workspace_bytes, ct_stream s);

/* grad = nabla R(x), curv = Huber curvature D_R(x) = 2 sum beta kappa kappa omega(x_j - x_n)
 * (factor 2 = separable quadratic surrogate split, R6).
 * kappa NULL = ones; curv NULL = skip. */
ct_status ct_reg_grad(const ct_geom* g, const ct_reg_desc* r, const float* x, const float* kappa, float* grad,
                      float* curv, ct_stream s);

/* Workspace bytes needed by oslalm_relaxed_solve for this geometry/params/dist. */
ct_status oslalm_workspace_size(const ct_geom* g, const oslalm_params* p, const ct_dist* dist, size_t* bytes);

/*
 * Run n_subiters sub-iterations of Algorithm 1 from state st:
 *   s  = rho (D_L x - h) + (1 - rho) g
 *   x+ = [x - (rho D_L + D_R)^{-1} (s + grad R(x))]_Omega
 *   zeta = M grad L_m(x+),  grad L_m(x) = A_m' W_m (A_m x - y_m)   (Eq. 36)
 *   g+ = rho/(rho+1) (alpha zeta + (1-alpha) g) + g/(rho+1)
 *   h+ = alpha (D_L x+ - zeta) + (1 - alpha) h
 *   rho <- rho_k(alpha) (Eq. 37), k = sub-iterations done
 * Subset m = k mod M (views v = m mod M).  y, w: full sinograms float[na][nt][ns]
 * (w NULL = ones).  d_l: D_L from ct_sqs_diag (required).  kappa NULL = ones.
 * x_ref / rms_per_iter (host double[], one entry per completed outer
 * iteration within this call) are optional; giving them synchronises.
 * dist != NULL shards each subset's views over the ranks (all ranks hold the
 * full volume): the partial back-projections are reduce-scattered by
 * z-slab (ncclReduceScatter, or grouped ncclReduce when nz % world != 0;
 * 2-D images: ncclAllReduce), the owner of each slab folds zeta into g, htilde
 * (lines 7-8) and updates x (lines 4-5) on its slab in one kernel, and x+ is
 * all-gathered (ncclAllGather / grouped ncclBroadcast) before its z-prefix is
 * rebuilt for the next forward.  grad R and D_R of the owner's slab of the new
 * x run on the communicator's side stream while the projections and the
 * reduction are in flight.  The last zeta of a call is folded and g, htilde
 * are all-gathered before the call returns, so a state handed back is always
 * complete and identical on every rank (resumable on any rank count).
 * 3-D: world <= nz (CT_E_CONFIG otherwise).
 * Single-GPU calls replay a cached CUDA graph of one sub-iteration.
 * Errors: CT_E_CONFIG (alpha not in [1,2), rho_fixed <= 0, M < 1 or M > na,
 * box_lo > box_hi, bad regulariser), CT_E_NOMEM (workspace), CT_E_NUMERIC
 * (non-finite x after the call), CT_E_CUDA, CT_E_NCCL.
 */
ct_status oslalm_relaxed_solve(const ct_geom* g, const float* y, const float* w, const ct_reg_desc* r,
                               const float* kappa, const float* d_l, const oslalm_params* p, oslalm_state* st,
                               int n_subiters, const float* x_ref, double* rms_per_iter, const ct_dist* dist,
                               void* workspace, size_t workspace_bytes, ct_stream s);

/*
 * Volume-domain (z-slab) decomposition:
 * rank p of `world` owns the planes [z0, z0 + nz) given by ct_zslab_range
 * (floor(p NZ / world) .. floor((p+1) NZ / world)) of x, g, htilde and D_L
 * (arrays of nz * ny * nx floats, boundary layout); every rank holds the full
 * y and w.  Per sub-iteration: slab x-update with one halo plane from each
 * neighbour, halo exchange (ncclSend/Recv), forward projection of the slab
 * for the subset's views, sum of the partial projections (ncclAllReduce of
 * V_m nt ns floats instead of the view decomposition's NX NY NZ) and the
 * weighted residual, back-projection onto the slab with the g / htilde
 * epilogue: every volume kernel works on 1/world of the volume.
 * One process per GPU: dist != NULL, nlocal = 1, the arrays of this rank.
 * One process driving all slabs on one device: dist == NULL, nlocal = world,
 * arrays indexed by rank (this is how the decomposition is tested on one GPU).
 * kappa is not supported (ones).  workspace[i]: >= the bytes of
 * oslalm_zslab_workspace_size for that slab, one buffer per local slab; slab
 * 0's buffer also holds the shared residual.  The state's k must agree across
 * slabs; k == 0 runs line 1 of Algorithm 1.  Errors as oslalm_relaxed_solve.
 */
ct_status ct_zslab_range(const ct_geom* g, int rank, int world, int* z0, int* nz);
ct_status oslalm_zslab_workspace_size(const ct_geom* g, const oslalm_params* p, int rank, int world, size_t* bytes);
/* D_L = diag(A'WA1) of the local slabs (same partial-projection sum). */
ct_status ct_sqs_diag_zslab(const ct_geom* g, const float* w, int nlocal, int world, const ct_dist* dist,
                            float* const* d_out, void* const* workspace, size_t workspace_bytes, ct_stream s);
ct_status oslalm_zslab_solve(const ct_geom* g, const float* y, const float* w, const ct_reg_desc* r,
                             const float* const* d_l, const oslalm_params* p, oslalm_state* st, int nlocal, int world,
                             int n_subiters, const ct_dist* dist, void* const* workspace, size_t workspace_bytes,
                             ct_stream s);

/* Same as oslalm_relaxed_solve (no x_ref/rms) but runs the sub-iterations
 * eagerly with CUDA events around each kernel and returns, in host
 * kernel_ms[4], the summed device time of (0) stencil + x-update, (1)
 * forward projection + residual, (2) back-projection (+ g/htilde epilogue),
 * (3) the rest (all-reduce, g/htilde update on the dist path, k advance).
 * Synchronises.  For measurement only. */
ct_status oslalm_profile(const ct_geom* g, const float* y, const float* w, const ct_reg_desc* r, const float* kappa,
                         const float* d_l, const oslalm_params* p, oslalm_state* st, int n_subiters,
                         const ct_dist* dist, void* workspace, size_t workspace_bytes, ct_stream s,
                         double* kernel_ms);

/* The weighted residual of the most recent sub-iteration of a solve (Eq. 36 /
 * Algorithm 1 line 6): r_out = W_m (A_m x+ - y_m) for the
 * views of subset m = (k - 1) mod M held by this rank (rank p of G: the
 * subset-local views p, p + G, ...), float[count][nt][ns].  k is the state's
 * counter after the oslalm_relaxed_solve call that ran sub-iteration k, with
 * the same g, p, dist and workspace (the residual lives in the workspace
 * until the next call).  For inspection and parity tests.  Errors:
 * CT_E_CONFIG (NULL, k < 1, params), CT_E_NOMEM (workspace), CT_E_CUDA. */
ct_status oslalm_residual(const ct_geom* g, const oslalm_params* p, const ct_dist* dist, int64_t k,
                          const void* workspace, size_t workspace_bytes, float* r_out, ct_stream s);

/* *d_count (device uint64) += number of nonzero entries of A on views v:
 * entry ((v,t,s),(i,j,k)) != 0 iff F1(s) > 0 and F2(k,t) > 0.
 * The projector's algorithmic FLOP count is 2 per nonzero. */
ct_status ct_count_nnz(const ct_geom* g, ct_views v, uint64_t* d_count, ct_stream s);

/* The units of SURVEY.md §8d's algorithmic FLOP figure for the projector pair on
 * views v: d_counts (device uint64[3]) += {nnz(A_v), in-cone voxel-view pairs
 * (voxels with at least one nonzero in the view), in-cone column-view pairs
 * (voxel columns with at least one nonzero in the view)}.  The bench's FLOP
 * count per projection is 2 nnz + 6 pairs + 150 columns (MACs, axial setup per
 * voxel, transaxial setup per column).  Errors as ct_count_nnz. */
ct_status ct_count_work(const ct_geom* g, ct_views v, uint64_t* d_counts, ct_stream s);

/* h = D_L x - htilde (Algorithm 1's h, for checkpoints and parity checks). */
ct_status oslalm_state_h(const ct_geom* g, const float* d_l, const oslalm_state* st, float* h_out, ct_stream s);

/* Eq. 37, pure host function: 1 if k == 0 else
 * pi/(alpha(k+1)) sqrt(1 - (pi/(2 alpha (k+1)))^2). */
double oslalm_rho(int64_t k, double alpha);

/* Host -> device copy of the views v of a sinogram-shaped array (y or w):
 * host and dev are both (na, nt, ns) float32 (host: pinned memory for an
 * asynchronous copy), and view rows start + i*stride, i < count, of host are
 * copied to the same rows of dev on stream s (one strided 2-D copy; other
 * rows untouched).  Lets a caller stream a subset's data ahead of the
 * sub-iteration that reads it (Algorithm 1 line 6 touches views of subset m
 * only).  Errors: CT_E_CONFIG (NULL), CT_E_SHAPE (views), CT_E_CUDA. */
ct_status ct_sino_upload(const ct_geom* g, const float* host, ct_views v, float* dev, ct_stream s);

/* Synchronise the stream and report deferred asynchronous errors. */
ct_status ct_sync(ct_stream s);

/* NCCL plumbing (one process per GPU).  The unique id (128 bytes) is created
 * on rank 0 and broadcast by the caller (e.g. torch.distributed).
 * ct_dist_create makes the communicator of rank `rank` of `world` on CUDA
 * device `device` (collective: every rank must call it), plus a
 * high-priority side stream and two events owned by the handle (the
 * stencil/all-reduce overlap of oslalm_relaxed_solve).  Errors: CT_E_CONFIG
 * (rank/world), CT_E_NCCL, CT_E_CUDA.  ct_dist_destroy frees all of it. */
ct_status ct_nccl_unique_id(unsigned char id[128]);
ct_status ct_dist_create(int rank, int world, const unsigned char id[128], int device, ct_dist** out);
/* Single-process emulation of a `world`-rank view-sharded solve on one device
 * (SURVEY.md §4 T4): passed as `dist`, the solver runs every rank's share of
 * each subset (rank p: the subset-local views p, p + world, ...; the device
 * picks them from its per-rank control block) into its own partial
 * back-projection, sums the partials in rank order (the reduce-scatter), has
 * each z-slab owner fold and update its slab (with halo planes from the
 * neighbouring slabs), and rebuilds the z-prefix of the whole x+ (the
 * all-gather is in place).  No NCCL.  ct_sqs_diag sums every rank's views the
 * same way; oslalm_residual returns rank 0's residual.  Errors: CT_E_CONFIG
 * (world outside [1, 64], device), CT_E_CUDA. */
ct_status ct_dist_create_local(int world, int device, ct_dist** out);
void ct_dist_destroy(ct_dist* d);

/* Number of this library's kernel launches since load (for bench accounting). */
int64_t ct_launch_count(void);

const char* ct_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CTRECON_H */
