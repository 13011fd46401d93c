"""GPU vs oracle parity on mid-size 3-D geometries that run the kernel instances
the BASELINE 3-D configs run (tests/geoms.py `mid`): two and four detector rows
per lane in the forward, 4-warp forward blocks (also inside the solve), the
z-prefix forward (the solver's), two 40-row passes and a ragged third z-chunk in
the back-projector, two update z-chunks with the per-row prefix exchange.

Tolerances (BASELINE.json north_star): projections 1e-4 relative L2; per-step
iterates x 1e-4, g / htilde 1e-3 (as tests/test_gpu_parity.py); GPU adjoint
identity 1e-5.  The weighted residual r = W(Ax - y) is compared with an error
normalised by ||W A x||: the residual inherits the projection's error times W,
and A x - y cancels most of A x.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import alg  # noqa: E402
from oracle import projector as P  # noqa: E402
from tests.geoms import MID_KINDS, fwd3_blocks, mid  # noqa: E402
from tests.problems import oracle_problem, rel, synthetic_problem  # noqa: E402


@pytest.fixture(scope="module")
def C():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1512_04564_b200 import ctrecon
    ctrecon.load()
    return ctrecon


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


@pytest.mark.parametrize("kind", MID_KINDS)
def test_mid_forward_back_zprefix_parity(C, kind):
    """ct_forward (direct z-loop), ct_forward_zprefix (the solver's z-prefix forward)
    and ct_back against the oracle over all views and a strided subset; GPU adjoint."""
    g = mid(kind)
    na = g["na"]
    nw, rpl = fwd3_blocks(g, na)
    assert rpl == (2 if g["nt"] <= 64 else 4) and (nw == 4) == (kind not in ("axial_mid",))
    rng = np.random.default_rng(31)
    x = rng.random(P.vol_shape(g))
    yv = rng.standard_normal(P.proj_shape(g, na))
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        xd = dev(x)
        ref = P.forward(g, x)
        pd = torch.empty(P.proj_shape(g, na), dtype=torch.float32, device="cuda")
        C.ct_forward(h, xd, C.views(0, 1, na), pd)
        pf = host(pd)
        assert rel(pf, ref) <= 1e-4, rel(pf, ref)
        ws = torch.empty(C.ct_zprefix_size(h), dtype=torch.uint8, device="cuda")
        pz = torch.empty_like(pd)
        C.ct_forward_zprefix(h, xd, C.views(0, 1, na), pz, ws)
        assert rel(host(pz), ref) <= 1e-4, rel(host(pz), ref)
        bd = torch.empty_like(xd)
        C.ct_back(h, dev(yv), C.views(0, 1, na), bd)
        bk = host(bd)
        assert rel(bk, P.back(g, yv)) <= 1e-4, rel(bk, P.back(g, yv))
        lhs, rhs = float(np.sum(pf * yv)), float(np.sum(x * bk))
        assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + abs(rhs)), (lhs, rhs)
        vv = (1, 3, (na - 1 + 2) // 3)
        ps = torch.empty(P.proj_shape(g, vv[2]), dtype=torch.float32, device="cuda")
        C.ct_forward_zprefix(h, xd, C.views(*vv), ps, ws)
        assert rel(host(ps), P.forward(g, x, vv)) <= 1e-4
        acc = dev(x)
        C.ct_back(h, ps, C.views(*vv), acc, scale=2.0, accumulate=True)
        assert rel(host(acc), x + 2.0 * P.back(g, host(ps), vv)) <= 1e-5
    finally:
        C.ct_geom_destroy(h)


@pytest.mark.parametrize("kind", MID_KINDS)
def test_mid_sqs_diag_parity(C, kind):
    g = mid(kind)
    rng = np.random.default_rng(32)
    w = rng.uniform(0.5, 2.0, P.proj_shape(g, g["na"]))
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        d = torch.empty(P.vol_shape(g), dtype=torch.float32, device="cuda")
        ws = torch.empty(37 * g["ns"] * g["nt"] * 4, dtype=torch.uint8, device="cuda")   # ragged chunks of views
        C.ct_sqs_diag(h, dev(w), d, ws)
        ref = P.back(g, w * P.forward(g, np.ones(P.vol_shape(g))))
        assert rel(host(d), ref) <= 1e-4, rel(host(d), ref)
    finally:
        C.ct_geom_destroy(h)


@pytest.mark.parametrize("kind", MID_KINDS)
def test_mid_solve_trace_and_residual(C, kind):
    """Algorithm 1 (M = 2) through the graph-replayed solve, the bench's launch path:
    x, g, htilde after sub-iterations 1, 2, 3, 5 against the oracle's trace, and the
    solver's own weighted residual of each of those sub-iterations (oslalm_residual)
    against W_m (A_m x+ - y_m) of the oracle."""
    from paper_1512_04564_b200.recon import Recon
    g = mid(kind)
    M = 2
    pb = synthetic_problem(g, M=M)
    prob = oracle_problem(pb)
    DL = pb["DL"]
    trace = {}
    alg.alg1(prob, pb["x0"], M, 1.999, 3, DL=DL, trace=trace)
    rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"])
    rec.compute_DL()
    assert rel(host(rec.dl), DL) <= 1e-4
    done = 0
    na = g["na"]
    for k in (1, 2, 3, 5):
        rec.run(k - done)
        done = k
        xo, go, ho = trace[k]
        assert rec.k == k
        assert rel(host(rec.x), xo) <= 1e-4, (k, rel(host(rec.x), xo))
        assert rel(host(rec.g), go) <= 1e-3, (k, rel(host(rec.g), go))
        assert rel(host(rec.htilde), DL * xo - ho) <= 1e-3, k
        m = (k - 1) % M
        views = alg.subset_views(na, M, m)
        r = torch.empty(P.proj_shape(g, views[2]), dtype=torch.float32, device="cuda")
        C.oslalm_residual(rec.h, rec.params, k, rec.ws, r)
        ax = P.forward(g, xo, views)
        wm = alg.subset_rows(pb["w"], na, M, m)
        ro = wm * (ax - alg.subset_rows(pb["y"], na, M, m))
        err = np.linalg.norm(host(r) - ro) / np.linalg.norm(wm * ax)
        assert err <= 1e-4, (k, err)
    rec.close()


@pytest.mark.parametrize("kind,nseg", [("helical_mid", 3), ("helical_rpl4", 2), ("axial_mid", 5),
                                       ("helical_thin", 4)])
def test_segmented_forward_parity(C, kind, nseg):
    """The segmented z-prefix forward (ct_geom_set_fwd_segments; automatic for c5-sized
    volumes): the wedge walked in nseg slab segments, tile-ordered blocks, segment sums
    added in order.  Against the oracle over all views (chunks of 128 views when na > 128)
    and a strided subset, against the unsegmented forward, and bitwise repeatable."""
    g = mid(kind)
    na = g["na"]
    rng = np.random.default_rng(41)
    x = rng.random(P.vol_shape(g))
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        assert C.ct_geom_fwd_segments(h, na) == 0      # mid-size volumes (< 256 x 256 columns): automatic = off
        xd = dev(x)
        ws0 = torch.empty(C.ct_zprefix_size(h), dtype=torch.uint8, device="cuda")
        p0 = torch.empty(P.proj_shape(g, na), dtype=torch.float32, device="cuda")
        C.ct_forward_zprefix(h, xd, C.views(0, 1, na), p0, ws0)
        C.ct_geom_set_fwd_segments(h, nseg)
        assert C.ct_geom_fwd_segments(h, na) == nseg
        ws = torch.empty(C.ct_zprefix_size(h), dtype=torch.uint8, device="cuda")
        assert ws.numel() > ws0.numel()
        ps = torch.empty_like(p0)
        C.ct_forward_zprefix(h, xd, C.views(0, 1, na), ps, ws)
        ref = P.forward(g, x)
        assert rel(host(ps), ref) <= 1e-4, rel(host(ps), ref)
        assert rel(host(ps), host(p0)) <= 1e-5
        ps2 = torch.empty_like(p0)
        C.ct_forward_zprefix(h, xd, C.views(0, 1, na), ps2, ws)
        assert torch.equal(ps, ps2)
        vv = (2, 3, (na - 2 + 2) // 3)
        pv = torch.empty(P.proj_shape(g, vv[2]), dtype=torch.float32, device="cuda")
        C.ct_forward_zprefix(h, xd, C.views(*vv), pv, ws)
        assert rel(host(pv), P.forward(g, x, vv)) <= 1e-4
        C.ct_geom_set_fwd_segments(h, -1)
        assert C.ct_geom_fwd_segments(h, na) == 0
    finally:
        C.ct_geom_destroy(h)


@pytest.mark.parametrize("kind,nseg", [("helical_mid", 3), ("helical_rpl4", 4)])
def test_segmented_solve_trace(C, kind, nseg):
    """Algorithm 1 (M = 2) with the segmented forward in the graph-replayed solve:
    x, g, htilde against the oracle's trace and the solver's residual against
    W_m (A_m x+ - y_m) of the oracle, as test_mid_solve_trace_and_residual."""
    from paper_1512_04564_b200.recon import Recon
    g = mid(kind)
    M = 2
    pb = synthetic_problem(g, M=M)
    prob = oracle_problem(pb)
    DL = pb["DL"]
    trace = {}
    alg.alg1(prob, pb["x0"], M, 1.999, 3, DL=DL, trace=trace)
    rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], fwd_segments=nseg)
    assert C.ct_geom_fwd_segments(rec.h, 200) == nseg
    rec.set_DL(DL)
    done = 0
    na = g["na"]
    for k in (1, 3, 5):
        rec.run(k - done)
        done = k
        xo, go, ho = trace[k]
        assert rel(host(rec.x), xo) <= 1e-4, (k, rel(host(rec.x), xo))
        assert rel(host(rec.g), go) <= 1e-3, (k, rel(host(rec.g), go))
        assert rel(host(rec.htilde), DL * xo - ho) <= 1e-3, k
        m = (k - 1) % M
        views = alg.subset_views(na, M, m)
        r = torch.empty(P.proj_shape(g, views[2]), dtype=torch.float32, device="cuda")
        C.oslalm_residual(rec.h, rec.params, k, rec.ws, r)
        ax = P.forward(g, xo, views)
        wm = alg.subset_rows(pb["w"], na, M, m)
        ro = wm * (ax - alg.subset_rows(pb["y"], na, M, m))
        err = np.linalg.norm(host(r) - ro) / np.linalg.norm(wm * ax)
        assert err <= 1e-4, (k, err)
    rec.close()


def test_automatic_segments_of_the_baseline_configs(C):
    """The library's automatic segment count for one subset of each BASELINE 3-D config
    (c5 16 for its 2.2 GB z-prefix, c4 3 and c3 8 from the 96 MB budget of partial
    sums) and off for the 2-D configs; forcing and resetting it."""
    from synth.configs import get_config
    want = {"c1": 0, "c2": 0, "c3": 8, "c4": 3, "c5": 16}
    for name, n in want.items():
        cfg = get_config(name)
        g, M = cfg["geom"], cfg["solver"]["M"]
        h = C.ct_geom_create(C.geom_desc(g))
        try:
            assert C.ct_geom_fwd_segments(h, (g["na"] + M - 1) // M) == n, name
            C.ct_geom_set_fwd_segments(h, 0)
            assert C.ct_geom_fwd_segments(h, (g["na"] + M - 1) // M) == 0
            C.ct_geom_set_fwd_segments(h, -1)
            assert C.ct_geom_fwd_segments(h, (g["na"] + M - 1) // M) == n
        finally:
            C.ct_geom_destroy(h)
