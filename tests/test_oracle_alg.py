"""Pins of the oracle iteration — CPU only.

Algorithm 1 has no external value to compare with for
M > 1 on the BASELINE configs; its parts are pinned here:
  P7a  Alg. 1 with M = 1 equals the literal Eq. 25 iteration with an explicit
       G^{1/2}, nu stays 0, for
       alpha in {1, 1.5, 1.999}, fixed rho and Eq. 37;
  P7b  alpha = 1: Alg. 1 == Alg. 2 == unrelaxed OS-LALM;
  P7d  Alg. 2 with M = 1 equals the literal Eq. 18 iteration (simple relaxation,
       PAPER.md:142-155) for alpha in {1.5, 1.999} (the alpha-dependent
       coefficients of its g recursion), fixed rho and Eq. 37;
  P7c  quadratic potential, M = 1: Alg. 1 converges to the dense PWLS
       minimiser (A'WA + H_R)^{-1}A'Wy; alpha = 1.999 gets there in fewer
       iterations than alpha = 1 (Theorem 2);
  P8   Eq. 37 values, subset partition, work accounting, feasibility;
  P9   M > 1: on a scan whose subsets are exact copies of each other (M turns,
       pitch 0) the ordered-subsets gradient is exact, and Alg. 1 / Alg. 2
       with M subsets equal the M = 1 iterations sub-iteration by
       sub-iteration (the subset loop, the M scaling, the rho counting and
       the line-1 subset are all exercised).
"""
import math

import numpy as np
import pytest

from oracle import alg, dense
from oracle import projector as P
from synth.configs import DIRECTIONS
from tests.geoms import tiny


def tiny_problem(kind="fan2d_arc", potential="hyperbola", beta=None, seed=0, **over):
    g = tiny(kind, **over)
    rng = np.random.default_rng(seed)
    shape = P.vol_shape(g)
    xt = 0.02 + 0.01 * rng.random(shape)
    ell = P.forward(g, xt)
    I0 = 1e4
    c = np.maximum(rng.poisson(I0 * np.exp(-ell)).astype(np.float64), 1.0)
    y = np.log(I0 / c)
    w = c / I0 * 10.0           # counts, rescaled to keep D_L O(1e2)
    n_dirs = 13 if g["dim"] == 3 else 4
    if beta is None:
        beta = 5.0
    betas = [beta] * n_dirs
    prob = alg.Problem(g, y, w, potential, 0.01, betas, n_dirs)
    x0 = np.clip(xt + 0.005 * rng.standard_normal(shape), 0, None)
    return prob, x0, xt


# ------------------------------------------------------------------ P8
def test_rho_eq37_values():
    # Direct evaluation of Eq. 37; values cross-checked
    # with SPEC.md:298-299 (0.97227 +- 1e-4, 0.72262 +- 1e-4) — see
    # tests/golden/rho_eq37.txt.
    golden = {}
    with open("tests/golden/rho_eq37.txt") as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, a, v = line.split()
                golden[(int(k), float(a))] = float(v)
    for (k, a), v in golden.items():
        assert abs(alg.rho_k(k, a) - v) <= 1e-6, (k, a)
    assert alg.rho_k(0, 1.999) == 1.0
    for a in (1.0, 1.3, 1.5, 1.999):
        seq = [alg.rho_k(k, a) for k in range(1, 3001)]
        assert all(s > 0 for s in seq) and all(b < c for b, c in zip(seq[1:], seq[:-1]))


def test_subsets_partition_gradient():
    prob, x0, _ = tiny_problem("helical_arc")
    M = 5
    full = prob.grad_L(x0)
    parts = sum(prob.grad_L_subset(x0, m, M) for m in range(M))
    assert np.allclose(parts, full, rtol=1e-12, atol=1e-12 * np.abs(full).max())
    views = sorted(v for m in range(M) for v in range(m, prob.g["na"], M))
    assert views == list(range(prob.g["na"]))


def test_work_accounting_and_feasibility():
    prob, x0, _ = tiny_problem("axial_flat")
    DL = prob.D_L()
    M = 3
    g, h = alg.alg1_init(prob, x0, M, DL)
    prob.n_fwd = prob.n_back = 0
    x, k = x0, 0
    for _ in range(7):
        x, g, h, k = alg.alg1_run(prob, x, g, h, k, 1, M, 1.999, DL)
        assert x.min() >= 0.0
    assert prob.n_fwd == 7 and prob.n_back == 7 and k == 7


def test_zero_data_zero_init_stays_zero():
    prob, x0, _ = tiny_problem()
    prob.y[:] = 0.0
    x = alg.alg1(prob, np.zeros_like(x0), 4, 1.999, 3)[0]
    assert np.all(x == 0.0)


# ------------------------------------------------------------------ P7a
@pytest.mark.parametrize("alpha", [1.0, 1.5, 1.999])
@pytest.mark.parametrize("rho_mode", ["fixed", "continuation"])
def test_alg1_M1_equals_literal_eq25(alpha, rho_mode):
    prob, x0, _ = tiny_problem("fan2d_arc", nx=8, ny=8, ns=16, na=12)
    g = prob.g
    DL = prob.D_L().ravel()
    A = dense.dense_A(g)
    sw = np.sqrt(prob.w.ravel())
    Aw, yw = sw[:, None] * A, sw * prob.y.ravel()       # Eq. 36 substitution
    n = 100
    rhos = [0.3] * n if rho_mode == "fixed" else [alg.rho_k(k, alpha) for k in range(n)]

    def psi_grad(x):
        return prob.reg(x.reshape(P.vol_shape(g)))[0].ravel()

    def psi_curv(x):
        return prob.reg(x.reshape(P.vol_shape(g)))[1].ravel()

    xs_lit, nus = dense.literal_eq25(Aw, yw, DL, x0.ravel(), alpha, rhos, psi_grad, psi_curv)
    xs_33 = dense.eq33(Aw, yw, DL, x0.ravel(), alpha, rhos, psi_grad, psi_curv)
    trace = {}
    alg.alg1(prob, x0, 1, alpha, n, DL=DL.reshape(x0.shape), rho_mode="continuation" if rho_mode != "fixed"
             else "fixed", rho_fixed=0.3, trace=trace)
    scale = max(np.abs(xs_lit[-1]).max(), 1e-30)
    for k in range(1, n + 1):
        assert np.max(np.abs(trace[k][0].ravel() - xs_lit[k])) <= 1e-10 * max(1.0, scale), k
        assert np.max(np.abs(xs_33[k] - xs_lit[k])) <= 1e-10 * max(1.0, scale), k
        assert np.all(nus[k] == 0.0)
    # the iteration moves (not a trivial fixed point)
    assert np.max(np.abs(xs_lit[-1] - xs_lit[0])) > 1e-4


# ------------------------------------------------------------------ P7d
@pytest.mark.parametrize("alpha", [1.5, 1.999])
@pytest.mark.parametrize("rho_mode", ["fixed", "continuation"])
def test_alg2_M1_equals_literal_eq18(alpha, rho_mode):
    prob, x0, _ = tiny_problem("fan2d_arc", nx=8, ny=8, ns=16, na=12)
    g = prob.g
    DL = prob.D_L()
    A = dense.dense_A(g)
    sw = np.sqrt(prob.w.ravel())
    Aw, yw = sw[:, None] * A, sw * prob.y.ravel()       # Eq. 36 substitution
    n = 100
    rhos = [0.3] * n if rho_mode == "fixed" else [alg.rho_k(k, alpha) for k in range(n)]

    def psi_grad(x):
        return prob.reg(x.reshape(P.vol_shape(g)))[0].ravel()

    def psi_curv(x):
        return prob.reg(x.reshape(P.vol_shape(g)))[1].ravel()

    xs = dense.literal_eq18(Aw, yw, DL.ravel(), x0.ravel(), alpha, rhos, psi_grad, psi_curv)
    scale = max(np.abs(xs[-1]).max(), 1.0)
    for k in (1, 2, 3, 10, 50, n):
        xa = alg.alg2(prob, x0, 1, alpha, k, DL=DL, rho_mode="continuation" if rho_mode != "fixed" else "fixed",
                      rho_fixed=0.3)[0]
        assert np.max(np.abs(xa.ravel() - xs[k])) <= 1e-10 * scale, k
    # and the early iterates differ from the proposed method's (Alg. 1) at alpha > 1 (both reach the
    # same fixed point later): the pin tells the two recursions apart
    x1 = alg.alg1(prob, x0, 1, alpha, 3, DL=DL, rho_mode="continuation" if rho_mode != "fixed" else "fixed",
                  rho_fixed=0.3)[0]
    assert np.max(np.abs(x1.ravel() - xs[3])) > 1e-3 * np.max(np.abs(xs[3] - xs[0]))
    assert np.max(np.abs(xs[-1] - xs[0])) > 1e-4


# ------------------------------------------------------------------ P7b
def test_alpha1_collapse():
    prob, x0, _ = tiny_problem("helical_arc")
    DL = prob.D_L()
    M, iters = 4, 15                    # 60 sub-iterations
    x1 = alg.alg1(prob, x0, M, 1.0, iters, DL=DL)[0]
    x2 = alg.alg2(prob, x0, M, 1.0, iters, DL=DL)[0]
    x3 = alg.os_lalm_unrelaxed(prob, x0, M, iters, DL=DL)
    nrm = np.linalg.norm(x3)
    assert np.linalg.norm(x1 - x3) <= 1e-12 * nrm
    assert np.linalg.norm(x2 - x3) <= 1e-12 * nrm
    # and relaxation really changes the iterates
    xr = alg.alg1(prob, x0, M, 1.999, iters, DL=DL)[0]
    assert np.linalg.norm(xr - x3) > 1e-6 * nrm


# ------------------------------------------------------------------ P7c
def test_converges_to_dense_pwls_minimiser():
    prob, x0, xt = tiny_problem("fan2d_arc", potential="quadratic", beta=0.5, nx=8, ny=8, ns=16, na=12)
    g = prob.g
    A = dense.dense_A(g)
    xhat = dense.dense_pwls_quadratic(A, prob.w.ravel(), prob.y.ravel(), P.vol_shape(g),
                                      DIRECTIONS[:prob.n_dirs], prob.betas)
    assert xhat.min() > 0.0          # box inactive at the minimiser
    DL = prob.D_L()
    reach = {}
    for alpha in (1.0, 1.999):
        x = x0.copy()
        gg, h = alg.alg1_init(prob, x, 1, DL)
        k = 0
        for it in range(20000):
            xn, gg, h, k = alg.alg1_run(prob, x, gg, h, k, 1, 1, alpha, DL, rho_mode="fixed", rho_fixed=0.5)
            err = np.linalg.norm(xn.ravel() - xhat) / np.linalg.norm(xhat)
            if alpha not in reach and err < 1e-6:
                reach[alpha] = it
            done = np.linalg.norm(xn - x) < 1e-13 * np.linalg.norm(x)
            x = xn
            if done:
                break
        assert np.linalg.norm(x.ravel() - xhat) <= 1e-8 * np.linalg.norm(xhat), alpha
    assert reach[1.999] < reach[1.0], reach


# ------------------------------------------------------------------ P7d (Alg. 2 / OS-SQS)
def test_os_sqs_monotone_descent_and_alg2_rho1_is_os_sqs():
    """OS-SQS with one subset is a majorize-minimize step (D_L majorizes A'WA,
    P5; the Huber D_R majorizes R, P6), so the PWLS cost (Eq. 34) cannot rise;
    Algorithm 2 with rho fixed to 1 (s = zeta) is OS-SQS with the subsets
    visited from M-1 (its zeta is the previous subset's gradient at x)."""
    prob, x0, _ = tiny_problem("helical_arc")
    DL = prob.D_L()
    x = x0.copy()
    c_prev = prob.cost(x)
    for _ in range(12):
        x = alg.os_sqs(prob, x, 1, 1, DL=DL)
        c = prob.cost(x)
        assert c <= c_prev * (1 + 1e-13), (c, c_prev)
        c_prev = c
    assert c_prev < 0.99 * prob.cost(x0)
    M, iters = 3, 4
    for alpha in (1.0, 1.999):       # g is unused when rho = 1
        x2 = alg.alg2(prob, x0, M, alpha, iters, DL=DL, rho_mode="fixed", rho_fixed=1.0)[0]
        xs = alg.os_sqs(prob, x0, M, iters, DL=DL, first=M - 1)
        assert np.linalg.norm(x2 - xs) <= 1e-12 * np.linalg.norm(xs), alpha
    # a different visiting order gives different iterates (the pin is not vacuous)
    assert np.linalg.norm(alg.os_sqs(prob, x0, M, iters, DL=DL) - xs) > 1e-8 * np.linalg.norm(xs)


# ------------------------------------------------------------------ P9 (M > 1)
def repeated_turn_problem(kind, V0, M, seed=3):
    """A pitch-0 scan of M full turns with V0 views per turn (na = M V0,
    gcd(M, V0) = 1): view v sits at angle 360 v / V0, so the views of every
    subset m = {v = m mod M} (PAPER.md:441-442 ordering, R4) are the V0
    distinct angles once each (subset partition R4), and the data of a view
    depend on its angle only.  Then M grad L_m(x) = grad L(x) exactly for every
    m: the ordered-subsets approximation of line 6 is exact, and Algorithm 1
    with M subsets must coincide, sub-iteration by sub-iteration, with
    Algorithm 1 with M = 1 on the same data (rho_k counts sub-iterations, R2;
    line 1 uses M grad L_{M-1} = grad L, R1)."""
    assert math.gcd(M, V0) == 1
    g = tiny(kind, na=M * V0, orbit_deg=360.0 * M, pitch=0.0)
    rng = np.random.default_rng(seed)
    shape = P.vol_shape(g)
    xt = 0.02 + 0.01 * rng.random(shape)
    ell = P.forward(g, xt)
    one = ell[:V0]                        # one turn; later turns repeat its angles
    I0 = 1e4
    c = np.maximum(rng.poisson(I0 * np.exp(-one)).astype(np.float64), 1.0)
    y = np.concatenate([np.log(I0 / c)] * M)
    w = np.concatenate([c / I0 * 10.0] * M)
    n_dirs = 13 if g["dim"] == 3 else 4
    prob = alg.Problem(g, y, w, "hyperbola", 0.01, [5.0] * n_dirs, n_dirs)
    x0 = np.clip(xt + 0.005 * rng.standard_normal(shape), 0, None)
    return prob, x0


@pytest.mark.parametrize("kind,V0,M", [("fan2d_arc", 8, 3), ("fan2d_flat", 7, 4), ("axial_flat", 5, 3)])
def test_os_with_exact_subsets_reduces_to_M1(kind, V0, M):
    prob, x0 = repeated_turn_problem(kind, V0, M)
    # the premise: every subset's scaled gradient is the full gradient
    gf = prob.grad_L(x0)
    for m in range(M):
        assert np.max(np.abs(M * prob.grad_L_subset(x0, m, M) - gf)) <= 1e-9 * np.max(np.abs(gf))
    DL = prob.D_L()
    K = 3
    for alpha in (1.0, 1.999):
        tr_M, tr_1 = {}, {}
        alg.alg1(prob, x0, M, alpha, K, DL=DL, trace=tr_M)
        alg.alg1(prob, x0, 1, alpha, K * M, DL=DL, trace=tr_1)
        for k in range(1, K * M + 1):
            for a, b in zip(tr_M[k], tr_1[k]):
                assert np.max(np.abs(a - b)) <= 1e-9 * max(np.max(np.abs(b)), 1e-30), (alpha, k)
    x_M, g_M = alg.alg2(prob, x0, M, 1.5, K, DL=DL)
    x_1, g_1 = alg.alg2(prob, x0, 1, 1.5, K * M, DL=DL)
    assert np.max(np.abs(x_M - x_1)) <= 1e-9 * np.max(np.abs(x_1))
    assert np.max(np.abs(g_M - g_1)) <= 1e-9 * np.max(np.abs(g_1))


def test_os_reduction_has_teeth():
    """On an ordinary one-turn scan the subsets differ, and the same comparison
    fails by orders of magnitude more than its tolerance."""
    prob, x0, _ = tiny_problem("fan2d_arc")
    DL = prob.D_L()
    tr_M, tr_1 = {}, {}
    alg.alg1(prob, x0, 3, 1.999, 1, DL=DL, trace=tr_M)
    alg.alg1(prob, x0, 1, 1.999, 3, DL=DL, trace=tr_1)
    d = np.max(np.abs(tr_M[3][0] - tr_1[3][0])) / np.max(np.abs(tr_1[3][0]))
    assert d > 1e-5, d
