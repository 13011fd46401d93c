"""Pins of the oracle regulariser (Eq. 35) — CPU."""
import itertools
import math

import numpy as np
import pytest

from oracle import projector as P
from synth.configs import DIRECTIONS, _geom

POTS = ["hyperbola", "fair", "quadratic", "qggmrf"]


def vol(nx, ny, nz, dz=1.0):
    return _geom(dim=3 if nz > 1 else 2, nx=nx, ny=ny, nz=nz, dz=dz)


def test_direction_table_matches_inputs_and_covers_26_neighbours():
    assert P.directions() == DIRECTIONS
    all_offsets = set()
    for d in DIRECTIONS:
        for sgn in (1, -1):
            all_offsets.add(tuple(sgn * c for c in d))
    expect = {o for o in itertools.product((-1, 0, 1), repeat=3) if o != (0, 0, 0)}
    assert all_offsets == expect and len(DIRECTIONS) == 13
    assert all(d[2] == 0 for d in DIRECTIONS[:4])


@pytest.mark.parametrize("pot", POTS)
def test_gradient_is_finite_difference_of_R(pot):
    g = vol(5, 4, 3)
    rng = np.random.default_rng(10)
    x = rng.random((3, 4, 5)) * 0.5
    kap = rng.uniform(0.5, 1.5, x.shape)
    betas = rng.uniform(0.5, 2.0, 13)
    delta = 0.3
    _, gr, _ = P.reg(g, pot, delta, betas, 13, x, kap)
    h = 1e-6
    fd = np.zeros_like(x)
    for idx in np.ndindex(x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd[idx] = (P.reg(g, pot, delta, betas, 13, xp, kap)[0] - P.reg(g, pot, delta, betas, 13, xm, kap)[0]) / (2 * h)
    assert np.max(np.abs(fd - gr)) <= 1e-6 * np.max(np.abs(gr))


@pytest.mark.parametrize("pot", POTS)
def test_huber_sqs_majorizes_R(pot):
    g = vol(5, 4, 3)
    rng = np.random.default_rng(11)
    x = rng.random((3, 4, 5))
    kap = rng.uniform(0.5, 1.5, x.shape)
    betas = rng.uniform(0.5, 2.0, 13)
    delta = 0.2
    R0, gr, cv = P.reg(g, pot, delta, betas, 13, x, kap)
    for scale in (1e-3, 0.1, 1.0, 5.0):
        for _ in range(25):
            z = x + scale * rng.standard_normal(x.shape)
            Rz = P.reg(g, pot, delta, betas, 13, z, kap)[0]
            Q = R0 + np.sum(gr * (z - x)) + 0.5 * np.sum(cv * (z - x) ** 2)
            assert Rz <= Q + 1e-12 * max(1.0, abs(Q))


@pytest.mark.parametrize("pot", POTS)
def test_constant_image_is_flat(pot):
    g = vol(4, 5, 3)
    x = np.full((3, 5, 4), 0.7)
    R, gr, _ = P.reg(g, pot, 0.1, np.ones(13), 13, x)
    assert R == 0.0 and np.all(gr == 0.0)


@pytest.mark.parametrize("pot", POTS)
def test_two_voxel_hand_expansion(pot):
    # 2x1 image (a, b), one direction (1,0,0), beta = 1.7, kappa = 1:
    # R = beta*phi(a-b), grad = beta*(phi'(a-b), -phi'(a-b)),
    # D_R = 2*beta*omega(a-b) on both voxels.
    g = vol(2, 1, 1)
    a, b, beta, d = 0.9, 0.25, 1.7, 0.4
    x = np.array([[[a, b]]])
    R, gr, cv = P.reg(g, pot, d, [beta], 1, x)
    t = a - b
    if pot == "quadratic":
        phi, dphi, om = t * t / 2, t, 1.0
    elif pot == "hyperbola":
        q = math.sqrt(1 + (t / d) ** 2)
        phi, dphi, om = d * d * (q - 1), t / q, 1 / q
    elif pot == "fair":
        phi, dphi, om = d * d * (abs(t) / d - math.log(1 + abs(t) / d)), t / (1 + abs(t) / d), 1 / (1 + abs(t) / d)
    else:   # q-GGMRF, p = 2, q = 1.2 (the default): phi = (t^2/2)/(1 + |t/d|^0.8)
        u = (abs(t) / d) ** 0.8
        phi = 0.5 * t * t / (1 + u)
        h = 1e-6       # phi' by a central difference of phi, omega = phi'/t
        dphi = (0.5 * (t + h) ** 2 / (1 + (abs(t + h) / d) ** 0.8) - 0.5 * (t - h) ** 2 / (1 + (abs(t - h) / d) ** 0.8)) / (2 * h)
        om = dphi / t
        assert np.isclose(R, beta * phi, rtol=1e-14)
        assert np.allclose(gr.ravel(), [beta * dphi, -beta * dphi], rtol=1e-8)
        assert np.allclose(cv.ravel(), [2 * beta * om] * 2, rtol=1e-8)
        return
    assert np.isclose(R, beta * phi, rtol=1e-14)
    assert np.allclose(gr.ravel(), [beta * dphi, -beta * dphi], rtol=1e-14)
    assert np.allclose(cv.ravel(), [2 * beta * om] * 2, rtol=1e-14)


def test_hyperbola_and_fair_at_delta():
    # hyperbola: phi'(delta) = delta/sqrt(2), omega(delta) = 1/sqrt(2);
    # Fair: phi'(delta) = delta/2 (e.g. t = delta = 10 -> 5), omega = 1/2.
    g = vol(2, 1, 1)
    for pot, dp, om in [("hyperbola", 1 / math.sqrt(2), 1 / math.sqrt(2)), ("fair", 0.5, 0.5)]:
        d = 10.0
        _, gr, cv = P.reg(g, pot, d, [1.0], 1, np.array([[[d, 0.0]]]))
        assert np.isclose(gr.ravel()[0], d * dp, rtol=1e-14)
        assert np.isclose(cv.ravel()[0], 2 * om, rtol=1e-14)


def test_chain_max_curvature_is_2_4_2():
    # quadratic potential (omega = 1): 1-D chain of 3, beta = 1 -> D_R = (2, 4, 2).
    g = vol(3, 1, 1)
    _, _, cv = P.reg(g, "quadratic", 1.0, [1.0], 1, np.random.default_rng(0).random((1, 1, 3)))
    assert np.allclose(cv.ravel(), [2.0, 4.0, 2.0])


def test_borders_drop_out_of_volume_pairs():
    # quadratic potential, unit betas: D_R = 2 * (number of in-volume neighbours).
    g = vol(3, 3, 3)
    _, _, cv = P.reg(g, "quadratic", 1.0, np.ones(13), 13, np.zeros((3, 3, 3)))
    assert cv[1, 1, 1] == 2 * 26 and cv[0, 0, 0] == 2 * 7 and cv[0, 1, 1] == 2 * 17
    g2 = vol(4, 4, 1)
    _, _, cv2 = P.reg(g2, "quadratic", 1.0, np.ones(4), 4, np.zeros((1, 4, 4)))
    assert cv2[0, 1, 1] == 2 * 8 and cv2[0, 0, 0] == 2 * 3


def test_sampled_reg_matches_full():
    g = vol(6, 5, 4)
    rng = np.random.default_rng(12)
    x = rng.random((4, 5, 6))
    kap = rng.uniform(0.5, 1.5, x.shape)
    _, gr, cv = P.reg(g, "hyperbola", 0.05, np.arange(1, 14) / 7.0, 13, x, kap)
    idx = rng.integers(0, x.size, 40)
    g2, c2 = P.reg_at(g, "hyperbola", 0.05, np.arange(1, 14) / 7.0, 13, x, idx, kap)
    assert np.allclose(g2, gr.ravel()[idx], rtol=1e-15) and np.allclose(c2, cv.ravel()[idx], rtol=1e-15)


def test_qggmrf_special_values():
    # p = 2 q-GGMRF (Thibault et al. 2007; PAPER.md:467 chest data):
    #   q = 2 reduces to the quadratic t^2/4 (u = 1 for every t);
    #   at t = delta (u = 1): phi = delta^2/4, phi' = delta (2 + q)/8, omega = (2 + q)/8;
    #   omega(0) = 1 like the other potentials (max curvature = 2 sum beta).
    g = vol(2, 1, 1)
    rng = np.random.default_rng(3)
    for t in rng.uniform(-3, 3, 5):
        R, gr, cv = P.reg(g, "qggmrf", 0.7, [1.0], 1, np.array([[[t, 0.0]]]), q=2.0)
        assert np.isclose(R, t * t / 4, rtol=1e-14) and np.isclose(gr.ravel()[0], t / 2, rtol=1e-14)
        assert np.isclose(cv.ravel()[0], 1.0, rtol=1e-14)
    d, q = 0.3, 1.3
    R, gr, cv = P.reg(g, "qggmrf", d, [1.0], 1, np.array([[[d, 0.0]]]), q=q)
    assert np.isclose(R, d * d / 4, rtol=1e-14)
    assert np.isclose(gr.ravel()[0], d * (2 + q) / 8, rtol=1e-14)
    assert np.isclose(cv.ravel()[0], 2 * (2 + q) / 8, rtol=1e-14)
    _, _, c0 = P.reg(g, "qggmrf", d, [1.0], 1, np.zeros((1, 1, 2)), q=q)
    assert np.allclose(c0, 2.0)


@pytest.mark.parametrize("pot", POTS)
def test_max_curvature_majorizes(pot):
    # curvature="max": D_R = 2 sum_n beta kappa kappa omega(0) = 2 sum beta kappa kappa, independent of x;
    # it is >= the Huber curvature (omega is largest at 0 for these potentials) and the SQS
    # inequality R(z) <= R(x) + <grad, z - x> + |z - x|^2_{D_R} / 2 still holds.
    g = vol(5, 4, 3)
    rng = np.random.default_rng(21)
    x = rng.random((3, 4, 5)) * 0.1
    kap = rng.uniform(0.5, 1.5, x.shape)
    betas = rng.uniform(0.5, 2.0, 13)
    R0, gr, ch = P.reg(g, pot, 0.05, betas, 13, x, kap)
    _, gm, cm = P.reg(g, pot, 0.05, betas, 13, x, kap, curvature="max")
    _, _, cq = P.reg(g, "quadratic", 0.05, betas, 13, rng.random(x.shape), kap)
    assert np.allclose(gm, gr, rtol=1e-15)
    assert np.allclose(cm, cq, rtol=1e-14)          # = the quadratic potential's (omega = 1) curvature
    assert np.all(cm >= ch * (1 - 1e-14))
    for _ in range(5):
        z = x + 0.05 * rng.standard_normal(x.shape)
        Rz = P.reg(g, pot, 0.05, betas, 13, z, kap)[0]
        Q = R0 + np.sum(gr * (z - x)) + 0.5 * np.sum(cm * (z - x) ** 2)
        assert Rz <= Q + 1e-12 * max(1.0, abs(Q))


def test_kappa_weights_closed_forms():
    # W = I gives kappa = 1; W = c I gives kappa = sqrt(c) (constant factors
    # cancel); voxels no ray reaches (0/0) get 1.  A voxel-dependent W changes kappa.
    from oracle import alg
    from tests.geoms import tiny
    g = tiny("helical_arc")
    shp = P.proj_shape(g, g["na"])
    k1 = alg.kappa_weights(g, np.ones(shp))
    assert np.allclose(k1, 1.0, rtol=1e-13)
    kc = alg.kappa_weights(g, 2.5 * np.ones(shp))
    assert np.allclose(kc, math.sqrt(2.5), rtol=1e-13)
    w = np.random.default_rng(4).uniform(0.5, 2.0, shp)
    kw = alg.kappa_weights(g, w)
    assert np.all(kw > math.sqrt(0.5) - 1e-12) and np.all(kw < math.sqrt(2.0) + 1e-12)
    assert np.std(kw) > 1e-3
