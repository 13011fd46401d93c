"""ORACLE (test infrastructure): the relaxed OS-LALM iteration in float64.

Algorithm 1 of PAPER.md:333-348 written out step by step in the paper's
notation, on top of the SF projector (oracle.projector) with the CT
substitution of Eq. 36 applied implicitly:
    grad L_m(x) = A_m' W_m (A_m x - y_m),   D_L = diag(A' W A 1).
Readings:
  R1  init "zeta = g = M grad L_M(x)" uses the LAST subset (0-based M-1).
  R2  sub-iteration j (1-based, global) uses rho_{j-1} for s and g+, then
      sets rho = rho_j (Eq. 37 with k = number of sub-iterations done).
  R4  subset m holds views v = m (mod M); visited m = 0..M-1.
  R11 Omega = {x >= 0}.   R12 zero denominator keeps x_j.
"""
import math

import numpy as np

from . import projector as P


def rho_k(k, alpha):
    """Eq. 37: rho_0 = 1, else
    pi/(alpha(k+1)) * sqrt(1 - (pi/(2 alpha (k+1)))^2)."""
    if k == 0:
        return 1.0
    a = math.pi / (alpha * (k + 1))
    return a * math.sqrt(1.0 - (math.pi / (2.0 * alpha * (k + 1))) ** 2)


def subset_views(na, M, m):
    """Views v = m (mod M): (start, stride, count) (reading R4)."""
    return (m, M, (na - m + M - 1) // M)


def subset_rows(arr, na, M, m):
    st, sd, cnt = subset_views(na, M, m)
    return arr[st::sd][:cnt]


class Problem:
    """PWLS CT problem of Eq. 34 with R of Eq. 35."""

    def __init__(self, geom, y, w, potential, delta, betas, n_dirs, kappa=None, q=1.2, curvature="huber"):
        self.g = geom
        self.y = np.asarray(y, dtype=np.float64)
        self.w = np.asarray(w, dtype=np.float64)
        self.potential = potential
        self.delta = float(delta)
        self.betas = list(betas)
        self.n_dirs = int(n_dirs)
        self.kappa = kappa
        self.q = float(q)                # q-GGMRF exponent (potential "qggmrf")
        self.curvature = curvature       # D_R: "huber" or "max"
        self.n_fwd = 0   # work accounting ("only once per iteration")
        self.n_back = 0

    def reg(self, x):
        _, gr, cv = P.reg(self.g, self.potential, self.delta, self.betas, self.n_dirs, x, self.kappa, q=self.q,
                          curvature=self.curvature)
        return gr, cv

    def reg_value(self, x):
        v, _, _ = P.reg(self.g, self.potential, self.delta, self.betas, self.n_dirs, x, self.kappa, q=self.q,
                        want_grad=False, want_curv=False)
        return v

    def grad_L_subset(self, x, m, M):
        """grad L_m(x) = A_m' W_m (A_m x - y_m) for subset m of M."""
        na = self.g["na"]
        views = subset_views(na, M, m)
        Ax = P.forward(self.g, x, views)
        self.n_fwd += 1
        r = subset_rows(self.w, na, M, m) * (Ax - subset_rows(self.y, na, M, m))
        self.n_back += 1
        return P.back(self.g, r, views)

    def grad_L(self, x):
        return self.grad_L_subset(x, 0, 1)

    def D_L(self):
        """diag(A' W A 1) over all views, computed once."""
        ones = np.ones(P.vol_shape(self.g))
        return P.back(self.g, self.w * P.forward(self.g, ones))

    def cost(self, x):
        r = P.forward(self.g, x) - self.y
        return 0.5 * float(np.sum(self.w * r * r)) + self.reg_value(x)


def kappa_weights(g, w):
    """Resolution-uniformity weights kappa of Eq. 35 (PAPER.md:319-321 cites them;
    formula as SPEC.md:529-531 reads [fessler:96:srp]):
    kappa_j = sqrt([A'W1]_j / [A'1]_j), 0/0 = 1, over all views."""
    aw = P.back(g, np.asarray(w, dtype=np.float64))
    a1 = P.back(g, np.ones(P.proj_shape(g, g["na"])))
    out = np.ones_like(a1)
    pos = a1 > 0
    out[pos] = np.sqrt(aw[pos] / a1[pos])
    return out


def _x_update(x, s, gradR, denom):
    """x+ = [x - (rho D_L + D_R)^{-1}(s + grad R(x))]_Omega; zero denominator keeps x."""
    safe = np.where(denom > 0, denom, 1.0)
    xn = np.where(denom > 0, x - (s + gradR) / safe, x)
    return np.maximum(xn, 0.0)


def alg1_init(prob, x, M, DL, init_grad="last"):
    """Line 1 of Alg. 1: rho = 1, zeta = g = M grad L_M(x), h = D_L x - zeta."""
    if init_grad == "last":
        zeta = M * prob.grad_L_subset(x, M - 1, M)
    else:
        zeta = prob.grad_L(x)
    g = zeta.copy()
    h = DL * x - zeta
    return g, h


def alg1_run(prob, x, g, h, k, n_subiters, M, alpha, DL, rho_mode="continuation", rho_fixed=None,
             trace=None):
    """n_subiters sub-iterations of Alg. 1 (lines 4-9) from state (x, g, h, k).

    Returns (x, g, h, k).  `trace`, if a dict, receives copies after every
    sub-iteration keyed by the global sub-iteration count."""
    x = np.array(x, dtype=np.float64)
    for _ in range(n_subiters):
        m = k % M
        rho = rho_k(k, alpha) if rho_mode == "continuation" else float(rho_fixed)
        gradR, DR = prob.reg(x)
        s = rho * (DL * x - h) + (1.0 - rho) * g                            # line 4
        x_new = _x_update(x, s, gradR, rho * DL + DR)                       # line 5
        zeta = M * prob.grad_L_subset(x_new, m, M)                          # line 6
        g_new = rho / (rho + 1.0) * (alpha * zeta + (1.0 - alpha) * g) + g / (rho + 1.0)  # line 7
        h_new = alpha * (DL * x_new - zeta) + (1.0 - alpha) * h              # line 8
        x, g, h = x_new, g_new, h_new
        k += 1                                                              # line 9 (Eq. 37)
        if trace is not None:
            trace[k] = (x.copy(), g.copy(), h.copy())
    return x, g, h, k


def alg1(prob, x0, M, alpha, iters, DL=None, rho_mode="continuation", rho_fixed=None, init_grad="last",
         trace=None):
    """Algorithm 1 (proposed relaxed OS-LALM), `iters` outer iterations."""
    if DL is None:
        DL = prob.D_L()
    x = np.array(x0, dtype=np.float64)
    g, h = alg1_init(prob, x, M, DL, init_grad)
    x, g, h, k = alg1_run(prob, x, g, h, 0, iters * M, M, alpha, DL, rho_mode, rho_fixed, trace)
    return x, g, h


def alg2(prob, x0, M, alpha, iters, DL=None, rho_mode="continuation", rho_fixed=None):
    """Algorithm 2 (simple relaxed OS-LALM), no h."""
    if DL is None:
        DL = prob.D_L()
    x = np.array(x0, dtype=np.float64)
    zeta = M * prob.grad_L_subset(x, M - 1, M)
    g = zeta.copy()
    k = 0
    for _ in range(iters):
        for m in range(M):
            rho = rho_k(k, alpha) if rho_mode == "continuation" else float(rho_fixed)
            gradR, DR = prob.reg(x)
            s = rho * zeta + (1.0 - rho) * g
            x = _x_update(x, s, gradR, rho * DL + DR)
            zeta = M * prob.grad_L_subset(x, m, M)
            g = rho / (rho + 1.0) * (alpha * zeta + (1.0 - alpha) * g) + g / (rho + 1.0)
            k += 1
    return x, g


def os_lalm_unrelaxed(prob, x0, M, iters, DL=None, rho_mode="continuation", rho_fixed=None):
    """Unrelaxed OS-LALM of [nien:15:fxr] coded on its own terms:
    s = rho*zeta + (1-rho)*g;  x+ = [x - (rho D_L + D_R)^{-1}(s + grad R)]_+;
    zeta = M grad L_m(x+);  g = (rho*zeta + g)/(rho + 1).
    ("When alpha = 1, both algorithms revert to the unrelaxed OS-LALM".)"""
    if DL is None:
        DL = prob.D_L()
    x = np.array(x0, dtype=np.float64)
    zeta = M * prob.grad_L_subset(x, M - 1, M)
    g = zeta.copy()
    k = 0
    for _ in range(iters):
        for m in range(M):
            rho = rho_k(k, 1.0) if rho_mode == "continuation" else float(rho_fixed)
            gradR, DR = prob.reg(x)
            x = _x_update(x, rho * zeta + (1.0 - rho) * g, gradR, rho * DL + DR)
            zeta = M * prob.grad_L_subset(x, m, M)
            g = (rho * zeta + g) / (rho + 1.0)
            k += 1
    return x


def os_sqs(prob, x0, M, iters, DL=None, first=0):
    """OS-SQS [erdogan:99:osa] (the paper's conventional baseline):
    x+ = [x - (D_L + D_R)^{-1}(M grad L_m(x) + grad R(x))]_+, subsets visited
    cyclically starting at subset `first`."""
    if DL is None:
        DL = prob.D_L()
    x = np.array(x0, dtype=np.float64)
    for _ in range(iters):
        for mm in range(M):
            m = (first + mm) % M
            gradR, DR = prob.reg(x)
            x = _x_update(x, M * prob.grad_L_subset(x, m, M), gradR, DL + DR)
    return x
