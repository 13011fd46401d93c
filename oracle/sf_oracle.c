/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header or
 * constant generator with paper_1512_04564_b200/ (the CUDA path).
 *
 * Plain float64 CPU implementation of
 *   - the separable-footprint (SF) projector pair A, A' exactly as defined in
 *     SURVEY.md 8c.1 (the paper only cites its projector, PAPER.md:315
 *     [long:10:3fa]; DESIGN.md "Readings" R15), and
 *   - the edge-preserving regulariser R(x) of PAPER.md:316-321 (Eq. 35), its
 *     gradient and the Huber curvature D_R (factor 2 =
 *     De Pierro split, R6).
 *
 * Every projector entry comes from ONE function (sf_column + F1 + F2 + Lz)
 * used by both the forward (voxel-driven scatter, parallel over views) and
 * the back-projection (voxel-driven gather, parallel over voxel columns), so
 * A' is the exact transpose of A.  Loops run in a fixed order per output
 * element, so results do not depend on the OpenMP thread count.
 *
 * Built with gcc -O2 -fopenmp (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int dim, nx, ny, nz;
    double dx, dy, dz, ox, oy, oz;
    int arc, ns, nt;
    double ds, dt, off_s, off_t, dso, dsd;
    int na;
    double orbit_deg, orbit_start_deg, pitch, source_z0;
} og_geom;

typedef struct {
    double cb, sb, zs;      /* cos beta, sin beta, source z */
    double Sx, Sy;          /* source position (x, y) */
} og_view;

typedef struct {
    double tau[4];          /* sorted corner taus */
    double lxy;             /* transaxial amplitude */
    double mag;             /* axial magnification */
    int s_lo, s_hi;         /* candidate cell range (inclusive) */
} og_fp;

static const double OG_PI = 3.14159265358979323846;

/* ---- geometry (SURVEY.md 8c.1 "Coordinates") ---- */
static void og_view_setup(const og_geom* g, int v, og_view* vw) {
    double beta = g->orbit_start_deg * OG_PI / 180.0 + (g->orbit_deg * OG_PI / 180.0) * (double)v / (double)g->na;
    double table = g->pitch * g->nt * g->dt * g->dso / g->dsd;
    double zstep = table * (g->orbit_deg / 360.0) / (double)g->na;
    vw->cb = cos(beta);
    vw->sb = sin(beta);
    vw->zs = g->source_z0 + (double)v * zstep;
    vw->Sx = g->dso * vw->cb;
    vw->Sy = g->dso * vw->sb;
}

static double og_xc(const og_geom* g, int i) { return ((double)i - 0.5 * (g->nx - 1)) * g->dx + g->ox; }
static double og_yc(const og_geom* g, int j) { return ((double)j - 0.5 * (g->ny - 1)) * g->dy + g->oy; }
static double og_zc(const og_geom* g, int k) { return ((double)k - 0.5 * (g->nz - 1)) * g->dz + g->oz; }

static double og_delta(const og_geom* g) { return g->arc ? g->ds / g->dsd : g->ds; }

/* transaxial detector coordinate of an in-plane point: flat Dsd*b/a, arc atan2(b,a) */
static double og_tau(const og_geom* g, const og_view* vw, double px, double py) {
    double rx = px - vw->Sx, ry = py - vw->Sy;
    double a = -(rx * vw->cb + ry * vw->sb);      /* (P-S).e_c, e_c = -(cos,sin) */
    double b = -rx * vw->sb + ry * vw->cb;        /* (P-S).e_u, e_u = (-sin,cos) */
    return g->arc ? atan2(b, a) : g->dsd * b / a;
}

static double og_sigma(const og_geom* g, int s) {
    return ((double)s - 0.5 * (g->ns - 1) - g->off_s) * og_delta(g);
}

static double og_theta(const og_geom* g, int t) {
    return ((double)t - 0.5 * (g->nt - 1) - g->off_t) * g->dt;
}

static void og_sort4(double* t) {
    for (int a = 1; a < 4; a++) {
        double key = t[a];
        int b = a - 1;
        while (b >= 0 && t[b] > key) { t[b + 1] = t[b]; b--; }
        t[b + 1] = key;
    }
}

/* Footprint of voxel column (i, j) in view vw (SURVEY.md 8c.1 bullets 3-5). */
static void og_column(const og_geom* g, const og_view* vw, int i, int j, og_fp* fp) {
    double cx = og_xc(g, i), cy = og_yc(g, j);
    double hx = 0.5 * g->dx, hy = 0.5 * g->dy;
    fp->tau[0] = og_tau(g, vw, cx - hx, cy - hy);
    fp->tau[1] = og_tau(g, vw, cx + hx, cy - hy);
    fp->tau[2] = og_tau(g, vw, cx - hx, cy + hy);
    fp->tau[3] = og_tau(g, vw, cx + hx, cy + hy);
    og_sort4(fp->tau);
    /* L_xy = min(dx/|d_x|, dy/|d_y|), d = unit direction S -> column centre */
    double rx = cx - vw->Sx, ry = cy - vw->Sy;
    double rn = sqrt(rx * rx + ry * ry);
    double ux = fabs(rx / rn), uy = fabs(ry / rn);
    double lx = ux > 0.0 ? g->dx / ux : INFINITY;
    double ly = uy > 0.0 ? g->dy / uy : INFINITY;
    fp->lxy = lx < ly ? lx : ly;
    /* magnification: flat Dsd/a(c), arc Dsd/|c-S|_xy */
    double a = -(rx * vw->cb + ry * vw->sb);
    fp->mag = g->arc ? g->dsd / rn : g->dsd / a;
    double D = og_delta(g);
    double c0 = 0.5 * (g->ns - 1) + g->off_s;
    int lo = (int)floor(fp->tau[0] / D + c0 + 0.5) - 1;
    int hi = (int)floor(fp->tau[3] / D + c0 + 0.5) + 1;
    fp->s_lo = lo < 0 ? 0 : lo;
    fp->s_hi = hi > g->ns - 1 ? g->ns - 1 : hi;
}

/* Antiderivative of the unit-height trapezoid. */
static double og_trapT(const double* t, double tau, double eps) {
    double r1 = t[1] - t[0], r2 = t[3] - t[2];
    if (tau <= t[0]) return 0.0;
    double T = 0.0;
    if (r1 > eps) {
        double u = tau < t[1] ? tau : t[1];
        T += (u - t[0]) * (u - t[0]) / (2.0 * r1);
    }
    if (tau <= t[1]) return T;
    double u = tau < t[2] ? tau : t[2];
    T += u - t[1];
    if (tau <= t[2]) return T;
    if (r2 > eps) {
        double u2 = tau < t[3] ? tau : t[3];
        T += 0.5 * r2 - (t[3] - u2) * (t[3] - u2) / (2.0 * r2);
    }
    return T;
}

/* F1(s): mean of the trapezoid over cell s. */
static double og_F1(const og_geom* g, const og_fp* fp, int s) {
    double D = og_delta(g);
    double sg = og_sigma(g, s);
    double eps = 1e-12 * D;
    return (og_trapT(fp->tau, sg + 0.5 * D, eps) - og_trapT(fp->tau, sg - 0.5 * D, eps)) / D;
}

/* F2(k, t): overlap of the magnified voxel z-extent with row t, / dt. */
static double og_F2(const og_geom* g, const og_view* vw, const og_fp* fp, int k, int t) {
    double zk = og_zc(g, k);
    double tm = fp->mag * (zk - 0.5 * g->dz - vw->zs);
    double tp = fp->mag * (zk + 0.5 * g->dz - vw->zs);
    double th = og_theta(g, t);
    double lo = tm > th - 0.5 * g->dt ? tm : th - 0.5 * g->dt;
    double hi = tp < th + 0.5 * g->dt ? tp : th + 0.5 * g->dt;
    return hi > lo ? (hi - lo) / g->dt : 0.0;
}

/* candidate rows of voxel k (inclusive), widened by one */
static void og_rows(const og_geom* g, const og_view* vw, const og_fp* fp, int k, int* tlo, int* thi) {
    double zk = og_zc(g, k);
    double tm = fp->mag * (zk - 0.5 * g->dz - vw->zs);
    double tp = fp->mag * (zk + 0.5 * g->dz - vw->zs);
    double c0 = 0.5 * (g->nt - 1) + g->off_t;
    int lo = (int)floor(tm / g->dt + c0 + 0.5) - 1;
    int hi = (int)floor(tp / g->dt + c0 + 0.5) + 1;
    *tlo = lo < 0 ? 0 : lo;
    *thi = hi > g->nt - 1 ? g->nt - 1 : hi;
}

/* per-ray amplitude L_z(s, t) */
static double og_Lz(const og_geom* g, int s, int t) {
    double th = og_theta(g, t);
    if (g->arc) return sqrt(g->dsd * g->dsd + th * th) / g->dsd;
    double sg = og_sigma(g, s);
    return sqrt(g->dsd * g->dsd + sg * sg + th * th) / sqrt(g->dsd * g->dsd + sg * sg);
}

/* ---------------- forward: proj[vi][t][s] = sum_j a_ij x_j ---------------- */
void og_forward(const og_geom* g, const double* x, int vstart, int vstride, int vcount, double* proj) {
    int nt = g->dim == 3 ? g->nt : 1;
    int nz = g->dim == 3 ? g->nz : 1;
    size_t nxy = (size_t)g->nx * g->ny;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int vi = 0; vi < vcount; vi++) {
        og_view vw;
        og_view_setup(g, vstart + vi * vstride, &vw);
        double* out = proj + (size_t)vi * nt * g->ns;
        memset(out, 0, sizeof(double) * nt * g->ns);
        double F1[4096];
        for (int j = 0; j < g->ny; j++) {
            for (int i = 0; i < g->nx; i++) {
                og_fp fp;
                og_column(g, &vw, i, j, &fp);
                for (int s = fp.s_lo; s <= fp.s_hi; s++) F1[s - fp.s_lo] = og_F1(g, &fp, s);
                if (g->dim != 3) {
                    double xv = x[(size_t)j * g->nx + i];
                    for (int s = fp.s_lo; s <= fp.s_hi; s++) out[s] += fp.lxy * F1[s - fp.s_lo] * xv;
                    continue;
                }
                for (int k = 0; k < nz; k++) {
                    double xv = x[(size_t)k * nxy + (size_t)j * g->nx + i];
                    int tlo, thi;
                    og_rows(g, &vw, &fp, k, &tlo, &thi);
                    for (int t = tlo; t <= thi; t++) {
                        double f2 = og_F2(g, &vw, &fp, k, t);
                        if (f2 <= 0.0) continue;
                        for (int s = fp.s_lo; s <= fp.s_hi; s++) {
                            double f1 = F1[s - fp.s_lo];
                            if (f1 <= 0.0) continue;
                            out[(size_t)t * g->ns + s] += og_Lz(g, s, t) * fp.lxy * f1 * f2 * xv;
                        }
                    }
                }
            }
        }
    }
}

/* ---------------- back: x_out[j] = sum_i a_ij proj_i ---------------- */
void og_back(const og_geom* g, const double* proj, int vstart, int vstride, int vcount, double* x_out) {
    int nt = g->dim == 3 ? g->nt : 1;
    int nz = g->dim == 3 ? g->nz : 1;
    size_t nxy = (size_t)g->nx * g->ny;
    #pragma omp parallel for schedule(dynamic, 16)
    for (long col = 0; col < (long)nxy; col++) {
        int j = (int)(col / g->nx), i = (int)(col % g->nx);
        double F1[4096];
        for (int k = 0; k < nz; k++) x_out[(size_t)k * nxy + col] = 0.0;
        for (int vi = 0; vi < vcount; vi++) {
            og_view vw;
            og_view_setup(g, vstart + vi * vstride, &vw);
            const double* pv = proj + (size_t)vi * nt * g->ns;
            og_fp fp;
            og_column(g, &vw, i, j, &fp);
            for (int s = fp.s_lo; s <= fp.s_hi; s++) F1[s - fp.s_lo] = og_F1(g, &fp, s);
            if (g->dim != 3) {
                double acc = 0.0;
                for (int s = fp.s_lo; s <= fp.s_hi; s++) acc += fp.lxy * F1[s - fp.s_lo] * pv[s];
                x_out[col] += acc;
                continue;
            }
            for (int k = 0; k < nz; k++) {
                int tlo, thi;
                og_rows(g, &vw, &fp, k, &tlo, &thi);
                double acc = 0.0;
                for (int t = tlo; t <= thi; t++) {
                    double f2 = og_F2(g, &vw, &fp, k, t);
                    if (f2 <= 0.0) continue;
                    for (int s = fp.s_lo; s <= fp.s_hi; s++) {
                        double f1 = F1[s - fp.s_lo];
                        if (f1 <= 0.0) continue;
                        acc += og_Lz(g, s, t) * fp.lxy * f1 * f2 * pv[(size_t)t * g->ns + s];
                    }
                }
                x_out[(size_t)k * nxy + col] += acc;
            }
        }
    }
}

/* Sampled forward: out[q] = [A x]_(v[q], t[q], s[q]) computed one ray at a time. */
void og_forward_rays(const og_geom* g, const double* x, int n, const int* vv, const int* ss, const int* tt,
                     double* out) {
    int nz = g->dim == 3 ? g->nz : 1;
    size_t nxy = (size_t)g->nx * g->ny;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int q = 0; q < n; q++) {
        og_view vw;
        og_view_setup(g, vv[q], &vw);
        int s = ss[q], t = tt[q];
        double acc = 0.0;
        for (int j = 0; j < g->ny; j++) {
            for (int i = 0; i < g->nx; i++) {
                og_fp fp;
                og_column(g, &vw, i, j, &fp);
                if (s < fp.s_lo || s > fp.s_hi) continue;
                double f1 = og_F1(g, &fp, s);
                if (f1 <= 0.0) continue;
                if (g->dim != 3) { acc += fp.lxy * f1 * x[(size_t)j * g->nx + i]; continue; }
                for (int k = 0; k < nz; k++) {
                    double f2 = og_F2(g, &vw, &fp, k, t);
                    if (f2 <= 0.0) continue;
                    acc += og_Lz(g, s, t) * fp.lxy * f1 * f2 * x[(size_t)k * nxy + (size_t)j * g->nx + i];
                }
            }
        }
        out[q] = acc;
    }
}

/* Sampled back-projection at flat voxel indices idx[q] (k*nx*ny + j*nx + i). */
void og_back_voxels(const og_geom* g, const double* proj, int vstart, int vstride, int vcount, int n,
                    const int64_t* idx, double* out) {
    int nt = g->dim == 3 ? g->nt : 1;
    size_t nxy = (size_t)g->nx * g->ny;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int q = 0; q < n; q++) {
        int k = (int)(idx[q] / (int64_t)nxy);
        int col = (int)(idx[q] % (int64_t)nxy);
        int j = col / g->nx, i = col % g->nx;
        double acc = 0.0;
        for (int vi = 0; vi < vcount; vi++) {
            og_view vw;
            og_view_setup(g, vstart + vi * vstride, &vw);
            const double* pv = proj + (size_t)vi * nt * g->ns;
            og_fp fp;
            og_column(g, &vw, i, j, &fp);
            for (int s = fp.s_lo; s <= fp.s_hi; s++) {
                double f1 = og_F1(g, &fp, s);
                if (f1 <= 0.0) continue;
                if (g->dim != 3) { acc += fp.lxy * f1 * pv[s]; continue; }
                int tlo, thi;
                og_rows(g, &vw, &fp, k, &tlo, &thi);
                for (int t = tlo; t <= thi; t++) {
                    double f2 = og_F2(g, &vw, &fp, k, t);
                    if (f2 <= 0.0) continue;
                    acc += og_Lz(g, s, t) * fp.lxy * f1 * f2 * pv[(size_t)t * g->ns + s];
                }
            }
        }
        out[q] = acc;
    }
}

/* ---------------- regulariser (Eq. 35) ---------------- */
/* 13 directions, each unordered neighbour pair once; first four in-plane. */
static const int OG_DIRS[13][3] = {
    {1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, -1, 0},
    {0, 0, 1}, {1, 0, 1}, {-1, 0, 1}, {0, 1, 1}, {0, -1, 1},
    {1, 1, 1}, {-1, 1, 1}, {1, -1, 1}, {-1, -1, 1},
};

void og_directions(int* out39) { memcpy(out39, OG_DIRS, sizeof(OG_DIRS)); }

/* potential 0 = quadratic, 1 = hyperbola, 2 = Fair, 3 = q-GGMRF with p = 2
 * (Thibault et al. 2007, the chest experiment's regulariser):
 * phi(t) = (t^2/2) / (1 + |t/delta|^(2-q)); returns phi, phi', omega = phi'/t. */
static void og_pot(int pot, double delta, double q, double t, double* phi, double* dphi, double* om) {
    if (pot == 0) { *phi = 0.5 * t * t; *dphi = t; *om = 1.0; return; }
    if (pot == 1) {
        double r = sqrt(1.0 + (t / delta) * (t / delta));
        *phi = delta * delta * (r - 1.0);
        *dphi = t / r;
        *om = 1.0 / r;
        return;
    }
    if (pot == 3) {
        /* d/dt [t^2/2 / (1+u)], u = |t/delta|^(2-q):  t (2 + q u) / (2 (1+u)^2) */
        double u = pow(fabs(t) / delta, 2.0 - q);
        *phi = 0.5 * t * t / (1.0 + u);
        *om = (2.0 + q * u) / (2.0 * (1.0 + u) * (1.0 + u));
        *dphi = t * *om;
        return;
    }
    double a = fabs(t) / delta;
    *phi = delta * delta * (a - log1p(a));
    *dphi = t / (1.0 + a);
    *om = 1.0 / (1.0 + a);
}

/* curvature: D_R_j = 2 sum beta kappa kappa omega(x_j - x_n) (Huber, maxcurv = 0) or with
 * omega(0) = 1, the maximum curvature of every potential here (maxcurv = 1). */
static void og_reg_voxel(const og_geom* g, int pot, double delta, double q, int maxcurv, const double* beta,
                         int ndirs, const double* x, const double* kappa, int i, int j, int k, double* gr,
                         double* cv) {
    int nz = g->dim == 3 ? g->nz : 1;
    size_t nxy = (size_t)g->nx * g->ny;
    size_t me = (size_t)k * nxy + (size_t)j * g->nx + i;
    double kj = kappa ? kappa[me] : 1.0;
    double sg = 0.0, sc = 0.0;
    for (int d = 0; d < ndirs; d++) {
        for (int sgn = -1; sgn <= 1; sgn += 2) {
            int ni = i + sgn * OG_DIRS[d][0], nj = j + sgn * OG_DIRS[d][1], nk = k + sgn * OG_DIRS[d][2];
            if (ni < 0 || nj < 0 || nk < 0 || ni >= g->nx || nj >= g->ny || nk >= nz) continue;
            size_t nb = (size_t)nk * nxy + (size_t)nj * g->nx + ni;
            double kn = kappa ? kappa[nb] : 1.0;
            double phi, dphi, om;
            og_pot(pot, delta, q, x[me] - x[nb], &phi, &dphi, &om);
            sg += beta[d] * kj * kn * dphi;
            sc += 2.0 * beta[d] * kj * kn * (maxcurv ? 1.0 : om);
        }
    }
    *gr = sg;
    *cv = sc;
}

/* grad = nabla R(x), curv = Huber curvature D_R (may be NULL); returns R(x). */
double og_reg(const og_geom* g, int pot, double delta, double q, int maxcurv, const double* beta, int ndirs,
              const double* x, const double* kappa, double* grad, double* curv) {
    int nz = g->dim == 3 ? g->nz : 1;
    size_t nxy = (size_t)g->nx * g->ny;
    double val = 0.0;
    #pragma omp parallel for reduction(+ : val) schedule(static)
    for (int k = 0; k < nz; k++) {
        for (int j = 0; j < g->ny; j++) {
            for (int i = 0; i < g->nx; i++) {
                size_t me = (size_t)k * nxy + (size_t)j * g->nx + i;
                double gr, cv;
                og_reg_voxel(g, pot, delta, q, maxcurv, beta, ndirs, x, kappa, i, j, k, &gr, &cv);
                if (grad) grad[me] = gr;
                if (curv) curv[me] = cv;
                /* value: each unordered pair once (forward directions only) */
                double kj = kappa ? kappa[me] : 1.0;
                for (int d = 0; d < ndirs; d++) {
                    int ni = i + OG_DIRS[d][0], nj = j + OG_DIRS[d][1], nk = k + OG_DIRS[d][2];
                    if (ni < 0 || nj < 0 || nk < 0 || ni >= g->nx || nj >= g->ny || nk >= nz) continue;
                    size_t nb = (size_t)nk * nxy + (size_t)nj * g->nx + ni;
                    double kn = kappa ? kappa[nb] : 1.0;
                    double phi, dphi, om;
                    og_pot(pot, delta, q, x[me] - x[nb], &phi, &dphi, &om);
                    val += beta[d] * kj * kn * phi;
                }
            }
        }
    }
    return val;
}

/* regulariser gradient / curvature at sampled flat voxel indices */
void og_reg_at(const og_geom* g, int pot, double delta, double q, int maxcurv, const double* beta, int ndirs,
               const double* x, const double* kappa, int n, const int64_t* idx, double* grad, double* curv) {
    size_t nxy = (size_t)g->nx * g->ny;
    #pragma omp parallel for schedule(static)
    for (int e = 0; e < n; e++) {
        int k = (int)(idx[e] / (int64_t)nxy);
        int col = (int)(idx[e] % (int64_t)nxy);
        og_reg_voxel(g, pot, delta, q, maxcurv, beta, ndirs, x, kappa, col % g->nx, col / g->nx, k, &grad[e],
                     &curv[e]);
    }
}

/* thread count control for the determinism test */
#ifdef _OPENMP
#include <omp.h>
void og_set_threads(int n) { omp_set_num_threads(n); }
int og_max_threads(void) { return omp_get_max_threads(); }
#else
void og_set_threads(int n) { (void)n; }
int og_max_threads(void) { return 1; }
#endif
