"""GPU (CUDA path, through the C-ABI) vs oracle parity — needs a B200.

Tolerances (BASELINE.json north_star): projections 1e-4
relative L2, reconstructed images 1e-3 relative RMS after a fixed number of
iterations; per-step traces 1e-4; GPU adjoint identity 1e-5.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import alg  # noqa: E402
from oracle import projector as P  # noqa: E402
from tests.geoms import FINE_KINDS, KINDS, tiny  # noqa: E402
from tests.problems import config_problem, oracle_problem, rel, synthetic_problem  # noqa: E402


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


GEOMS = {k: tiny(k) for k in KINDS + FINE_KINDS}
GEOMS["c1"] = None  # filled lazily from synth


def geom_of(name):
    if name == "c1":
        from synth.configs import get_config
        return get_config("c1")["geom"]
    return GEOMS[name]


@pytest.mark.parametrize("name", KINDS + FINE_KINDS + ["c1"])
def test_forward_back_parity(C, name):
    g = geom_of(name)
    rng = np.random.default_rng(7)
    x = rng.random(P.vol_shape(g))
    cnt = g["na"]
    yv = rng.standard_normal(P.proj_shape(g, cnt))
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        xd = dev(x)
        pd = torch.empty(P.proj_shape(g, cnt), dtype=torch.float32, device="cuda")
        C.ct_forward(h, xd, C.views(0, 1, cnt), pd)
        pf = host(pd)
        ref = P.forward(g, x)
        assert rel(pf, ref) <= 1e-4, rel(pf, ref)
        bd = torch.empty_like(xd)
        C.ct_back(h, dev(yv), C.views(0, 1, cnt), bd)
        bk = host(bd)
        refb = P.back(g, yv)
        assert rel(bk, refb) <= 1e-4, rel(bk, refb)
        # GPU adjoint identity <Ax, y> = <x, A'y>
        lhs = float(np.sum(pf * yv))
        rhs = float(np.sum(x * bk))
        assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + abs(rhs)), (lhs, rhs)
        # a strided subset, scale and accumulate
        vv = (1, 3, (cnt - 1 + 2) // 3)
        ps = torch.empty(P.proj_shape(g, vv[2]), dtype=torch.float32, device="cuda")
        C.ct_forward(h, xd, C.views(*vv), ps)
        assert rel(host(ps), P.forward(g, x, vv)) <= 1e-4
        acc = dev(x)
        C.ct_back(h, ps, C.views(*vv), acc, scale=2.0, accumulate=True)
        assert rel(host(acc), x + 2.0 * P.back(g, host(ps), vv)) <= 1e-5
    finally:
        C.ct_geom_destroy(h)


@pytest.mark.parametrize("name", KINDS + FINE_KINDS)
def test_sqs_diag_parity(C, name):
    g = geom_of(name)
    rng = np.random.default_rng(8)
    w = rng.uniform(0.5, 2.0, P.proj_shape(g, g["na"]))
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        d = torch.empty(P.vol_shape(g), dtype=torch.float32, device="cuda")
        ws = torch.empty(3 * g["ns"] * (g["nt"] if g["dim"] == 3 else 1) * 4 + 7, dtype=torch.uint8,
                         device="cuda")   # 3 views per chunk: exercises chunking and a ragged tail
        C.ct_sqs_diag(h, dev(w), d, ws)
        ref = P.back(g, w * P.forward(g, np.ones(P.vol_shape(g))))
        assert rel(host(d), ref) <= 1e-4
    finally:
        C.ct_geom_destroy(h)


@pytest.mark.parametrize("pot", ["hyperbola", "fair", "quadratic", "qggmrf"])
@pytest.mark.parametrize("kind", ["fan2d_arc", "helical_arc"])
@pytest.mark.parametrize("use_kappa", [False, True])
@pytest.mark.parametrize("curvature", ["huber", "max"])
def test_reg_grad_parity(C, pot, kind, use_kappa, curvature):
    g = tiny(kind, nx=37, ny=21, nz=9) if kind == "helical_arc" else tiny(kind, nx=37, ny=21)
    rng = np.random.default_rng(9)
    x = 0.02 * rng.random(P.vol_shape(g))
    kap = rng.uniform(0.5, 1.5, x.shape) if use_kappa else None
    nd = 13 if g["dim"] == 3 else 4
    betas = list(rng.uniform(0.5, 2.0, nd))
    _, gr, cv = P.reg(g, pot, 0.01, betas, nd, x, kap, q=1.3, curvature=curvature)
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        gd = torch.empty(x.shape, dtype=torch.float32, device="cuda")
        cd = torch.empty_like(gd)
        C.ct_reg_grad(h, C.reg_desc(pot, 0.01, betas, nd, curvature, 1.3), dev(x), gd, cd,
                      kappa=dev(kap) if use_kappa else None)
        assert rel(host(gd), gr) <= 1e-5
        assert rel(host(cd), cv) <= 1e-5
    finally:
        C.ct_geom_destroy(h)


@pytest.mark.parametrize("delta", [1e-4, 1e-3, 10.0])
def test_reg_grad_hyperbola_delta_range(C, delta):
    """Hyperbola stencil from the near-TV (|t| ~ 0.02 >> delta) to the near-quadratic (delta = 10)
    regime.  The kernel's register window holds x/delta in float32, so t/delta
    carries an absolute rounding of ~ulp(|x|/delta): below delta ~ 1e-5 at |x| ~ 0.02 that exceeds
    the 1e-5 bar for pairs with |t| ~ delta (measured 2.9e-4 on D_R at delta = 1e-6; the UPD_RAW
    switch, exact t, avoids it but is slower).  The oracle gets the same float32-rounded x."""
    g = tiny("helical_arc", nx=37, ny=21, nz=9)
    rng = np.random.default_rng(11)
    x = (0.02 * rng.random(P.vol_shape(g))).astype(np.float32).astype(np.float64)
    betas = list(rng.uniform(0.5, 2.0, 13))
    _, gr, cv = P.reg(g, "hyperbola", delta, betas, 13, x, None)
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        gd = torch.empty(x.shape, dtype=torch.float32, device="cuda")
        cd = torch.empty_like(gd)
        C.ct_reg_grad(h, C.reg_desc("hyperbola", delta, betas, 13), dev(x), gd, cd)
        assert rel(host(gd), gr) <= 1e-5
        assert rel(host(cd), cv) <= 1e-5
        with pytest.raises(C.CtError):
            C.ct_reg_grad(h, C.reg_desc("hyperbola", 1e-20, betas, 13), dev(x), gd, cd)
    finally:
        C.ct_geom_destroy(h)


def _gpu_recon(pb, dl=None):
    from paper_1512_04564_b200.recon import Recon
    r = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"])
    if dl is None:
        r.compute_DL()
    else:
        r.set_DL(dl)
    return r


@pytest.mark.parametrize("kind", KINDS + FINE_KINDS)
def test_solve_trace_matches_oracle(C, kind):
    """Per-step trace: x, g and htilde after sub-iterations 1, 2, 3, M, 2M."""
    pb = synthetic_problem(tiny(kind), M=3)
    prob = oracle_problem(pb)
    DL = pb["DL"]
    trace = {}
    alg.alg1(prob, pb["x0"], 3, 1.999, 2, DL=DL, trace=trace)
    rec = _gpu_recon(pb)
    assert rel(host(rec.dl), DL) <= 1e-4
    done = 0
    for k in (1, 2, 3, 6):
        rec.run(k - done)
        done = k
        xo, go, ho = trace[k]
        assert rec.k == k
        assert rel(host(rec.x), xo) <= 1e-4, (k, rel(host(rec.x), xo))
        assert rel(host(rec.g), go) <= 1e-3, (k, rel(host(rec.g), go))
        assert rel(host(rec.htilde), DL * xo - ho) <= 1e-3, k
    rec.close()


@pytest.mark.parametrize("kind", ["helical_arc", "fan2d_arc"])
def test_alg2_simple_and_os_sqs_match_oracle(C, kind):
    """Algorithm 2 (variant SIMPLE) and OS-SQS (SIMPLE with rho fixed
    to 1) through the C-ABI against the oracle's alg2 / os_sqs."""
    pb = synthetic_problem(tiny(kind), M=3)
    prob = oracle_problem(pb)
    DL = pb["DL"]
    M, iters = 3, 2
    xo, go = alg.alg2(prob, pb["x0"], M, 1.999, iters, DL=DL)
    rec = _gpu_recon(dict(pb, solver=dict(pb["solver"], variant="simple")), dl=DL)
    rec.run(M * iters)
    assert rel(host(rec.x), xo) <= 1e-4
    assert rel(host(rec.g), go) <= 1e-3
    rec.close()
    xs = alg.os_sqs(prob, pb["x0"], M, iters, DL=DL, first=M - 1)
    rec = _gpu_recon(dict(pb, solver=dict(pb["solver"], variant="simple", rho_mode="fixed", rho_fixed=1.0)), dl=DL)
    rec.run(M * iters)
    assert rel(host(rec.x), xs) <= 1e-4
    rec.close()


def test_alpha1_alg1_equals_alg2_on_gpu(C):
    """alpha = 1: both recursions revert to the unrelaxed OS-LALM."""
    pb = synthetic_problem(tiny("helical_arc"), M=3, alpha=1.0)
    outs = []
    for variant in ("proposed", "simple"):
        rec = _gpu_recon(dict(pb, solver=dict(pb["solver"], variant=variant)), dl=pb["DL"])
        rec.run(7)
        outs.append((host(rec.x), host(rec.g)))
        rec.close()
    assert rel(outs[1][0], outs[0][0]) <= 1e-5
    assert rel(outs[1][1], outs[0][1]) <= 1e-5


@pytest.mark.parametrize("kind", ["helical_arc", "fan2d_arc"])
def test_qggmrf_max_curvature_solve_matches_oracle(C, kind):
    """q-GGMRF potential with the maximum-curvature D_R
    through the solver against the oracle's Algorithm 1."""
    pb = synthetic_problem(tiny(kind), M=3)
    pb["reg"] = dict(pb["reg"], potential="qggmrf", q=1.2, curvature="max")
    prob = oracle_problem(pb)
    xo, go, ho = alg.alg1(prob, pb["x0"], 3, 1.999, 2, DL=pb["DL"])
    rec = _gpu_recon(pb, dl=pb["DL"])
    rec.run(6)
    assert rel(host(rec.x), xo) <= 1e-4
    assert rel(host(rec.g), go) <= 1e-3
    rec.close()


@pytest.mark.parametrize("name", KINDS)
def test_kappa_weights_parity_and_kappa_solve(C, name):
    """ct_kappa_weights (SPEC.md:529-531 reading of P:321's kappa) against the oracle,
    with a workspace that forces chunking; then Algorithm 1 with that kappa."""
    g = geom_of(name)
    pb = synthetic_problem(g, M=3)
    ko = alg.kappa_weights(g, pb["w"])
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        kd = torch.empty(P.vol_shape(g), dtype=torch.float32, device="cuda")
        nvox = int(np.prod(P.vol_shape(g)))
        per_view = g["ns"] * (g["nt"] if g["dim"] == 3 else 1) * 4
        ws = torch.empty(((nvox * 4 + 255) // 256) * 256 + 3 * per_view + 5, dtype=torch.uint8, device="cuda")
        C.ct_kappa_weights(h, dev(pb["w"]), kd, ws)
        assert rel(host(kd), ko) <= 1e-5
    finally:
        C.ct_geom_destroy(h)
    prob = oracle_problem(pb)
    prob.kappa = ko
    xo = alg.alg1(prob, pb["x0"], 3, 1.999, 2, DL=pb["DL"])[0]
    from paper_1512_04564_b200.recon import Recon
    rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], kappa=host(kd))
    rec.set_DL(pb["DL"])
    rec.run(6)
    assert rel(host(rec.x), xo) <= 1e-4
    rec.close()


@pytest.mark.parametrize("name", ["fan2d_arc", "fan2d_flat", "axial_flat", "axial_arc", "c1"])
def test_fbp_parity(C, name):
    """ct_fbp (FBP / FDK initialiser) against oracle/fbp.py on the
    analytic line integrals of the config's random-ellipse phantom."""
    from oracle import fbp as F
    from synth.phantom import analytic_sinogram, sample_ellipsoids
    g = tiny("axial_flat", det="arc", ds=0.018 * 180.0 / 1.0) if name == "axial_arc" else geom_of(name)
    ells = sample_ellipsoids(g, 6, 11)
    sino = analytic_sinogram(g, ells, sub_s=1, sub_t=1).numpy()
    ref = F.fbp(g, sino)
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        out = torch.empty(P.vol_shape(g), dtype=torch.float32, device="cuda")
        ws = torch.empty(sino.size * 4, dtype=torch.uint8, device="cuda")
        C.ct_fbp(h, dev(sino), out, ws)
        assert rel(host(out), ref) <= 1e-4, rel(host(out), ref)
    finally:
        C.ct_geom_destroy(h)


def test_fbp_rejects_helical(C):
    g = tiny("helical_arc")
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        out = torch.empty(P.vol_shape(g), dtype=torch.float32, device="cuda")
        ws = torch.empty(g["na"] * g["nt"] * g["ns"] * 4, dtype=torch.uint8, device="cuda")
        with pytest.raises(C.CtError):
            C.ct_fbp(h, torch.zeros(P.proj_shape(g, g["na"]), device="cuda"), out, ws)
    finally:
        C.ct_geom_destroy(h)


def test_c1_full_solve_matches_oracle(C):
    """BASELINE configs[0]: 128^2 fan, 180 views, M = 4, 20 iterations, alpha = 1.999."""
    pb = config_problem("c1")
    prob = oracle_problem(pb)
    M, iters, a = pb["solver"]["M"], pb["solver"]["iters"], pb["solver"]["alpha"]
    xo = alg.alg1(prob, pb["x0"], M, a, iters, DL=pb["DL"])[0]
    rec = _gpu_recon(pb)
    rec.run(M * iters)
    xg = host(rec.x)
    rms = math.sqrt(np.mean((xg - xo) ** 2)) / math.sqrt(np.mean(xo ** 2))
    assert rms <= 1e-3, rms
    assert xg.min() >= 0.0
    rec.close()


def test_alpha1_and_fixed_rho_and_full_init(C):
    pb = synthetic_problem(tiny("axial_flat"), M=4, alpha=1.0)
    pb["solver"].update(rho_mode="fixed", rho_fixed=0.3, init_grad="full")
    prob = oracle_problem(pb)
    x = pb["x0"].copy()
    g, h = alg.alg1_init(prob, x, 4, pb["DL"], init_grad="full")
    xo, go, ho, k = alg.alg1_run(prob, x, g, h, 0, 10, 4, 1.0, pb["DL"], rho_mode="fixed", rho_fixed=0.3)
    rec = _gpu_recon(pb)
    rec.run(10)
    assert rel(host(rec.x), xo) <= 1e-4
    rec.close()


def test_ragged_subsets_and_resume(C):
    """M does not divide na (ragged last subsets); state resumes across calls."""
    g = tiny("helical_arc", na=41)
    pb = synthetic_problem(g, M=4)
    prob = oracle_problem(pb)
    trace = {}
    alg.alg1(prob, pb["x0"], 4, 1.999, 3, DL=pb["DL"], trace=trace)
    rec = _gpu_recon(pb)
    for n in (1, 4, 2, 5):
        rec.run(n)
    assert rec.k == 12
    assert rel(host(rec.x), trace[12][0]) <= 1e-4
    rec.close()


def test_zero_data_zero_init_stays_zero(C):
    pb = synthetic_problem(tiny("fan2d_arc"))
    pb["y"] = np.zeros_like(pb["y"])
    pb["x0"] = np.zeros_like(pb["x0"])
    rec = _gpu_recon(pb)
    rec.run(7)
    assert float(rec.x.abs().max()) == 0.0
    rec.close()


def test_errors_have_no_side_effects(C):
    g = tiny("fan2d_arc")
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        x = torch.zeros(P.vol_shape(g), dtype=torch.float32, device="cuda")
        p = torch.full(P.proj_shape(g, 2), 7.0, dtype=torch.float32, device="cuda")
        with pytest.raises(C.CtError) as e:
            C.ct_forward(h, x, C.views(g["na"] - 1, 1, 2), p)   # runs past the last view
        assert e.value.status == C.CT_E_SHAPE
        assert float(p.min()) == 7.0
        pb = synthetic_problem(g)
        from paper_1512_04564_b200.recon import Recon
        for bad in (dict(alpha=2.0), dict(alpha=0.5), dict(M=0), dict(M=g["na"] + 1)):
            s = dict(pb["solver"], **bad)
            with pytest.raises(C.CtError) as e:
                Recon(g, pb["reg"], s, pb["y"], pb["w"], pb["x0"])
            assert e.value.status == C.CT_E_CONFIG
        bad_reg = dict(pb["reg"], delta=0.0)
        r = Recon(g, pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"])
        r.compute_DL()
        r.reg = C.reg_desc("hyperbola", 0.0, bad_reg["betas"], 4)
        x_before = r.x.clone()
        with pytest.raises(C.CtError) as e:
            r.run(3)
        assert e.value.status == C.CT_E_CONFIG and r.k == 0 and torch.equal(r.x, x_before)
        r.close()
        bad_geom = dict(g, dso=5.0, dsd=9.0)
        with pytest.raises(C.CtError) as e:
            C.ct_geom_create(C.geom_desc(bad_geom))
        assert e.value.status == C.CT_E_CONFIG
        for bad_g in (tiny("helical_arc", nz=1537), tiny("helical_arc", nx=70000, ny=70000)):
            with pytest.raises(C.CtError) as e:
                C.ct_geom_create(C.geom_desc(bad_g))
            assert e.value.status == C.CT_E_CONFIG
        # variant / curvature / q-GGMRF exponent outside their ranges, before any launch
        for bad in (dict(variant="bogus"),):
            with pytest.raises(ValueError):
                Recon(g, pb["reg"], dict(pb["solver"], **bad), pb["y"], pb["w"], pb["x0"]).run(1)
        r = Recon(g, pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"])
        r.compute_DL()
        x_before = r.x.clone()
        for reg in (C.reg_desc("qggmrf", 0.01, pb["reg"]["betas"], 4, "huber", 2.5),
                    C.reg_desc("qggmrf", 0.01, pb["reg"]["betas"], 4, "huber", 0.5)):
            r.reg = reg
            with pytest.raises(C.CtError) as e:
                r.run(2)
            assert e.value.status == C.CT_E_CONFIG and r.k == 0 and torch.equal(r.x, x_before)
        r.reg = C.reg_desc("hyperbola", 0.01, pb["reg"]["betas"], 4)
        r.reg.curvature = 7
        with pytest.raises(C.CtError) as e:
            r.run(2)
        assert e.value.status == C.CT_E_CONFIG and r.k == 0
        r.params.variant = 5
        r.reg = C.reg_desc("hyperbola", 0.01, pb["reg"]["betas"], 4)
        with pytest.raises(C.CtError) as e:
            r.run(2)
        assert e.value.status == C.CT_E_CONFIG and r.k == 0
        r.close()
        # FBP needs a 360-degree orbit
        hs = C.ct_geom_create(C.geom_desc(dict(g, orbit_deg=200.0)))
        try:
            ws = torch.empty(g["na"] * g["ns"] * 4, dtype=torch.uint8, device="cuda")
            with pytest.raises(C.CtError) as e:
                C.ct_fbp(hs, torch.zeros(P.proj_shape(g, g["na"]), device="cuda"), x, ws)
            assert e.value.status == C.CT_E_CONFIG
        finally:
            C.ct_geom_destroy(hs)
        # empty view descriptor is a no-op
        C.ct_forward(h, x, C.views(0, 1, 0), p)
        assert float(p.min()) == 7.0
    finally:
        C.ct_geom_destroy(h)


def test_deterministic_repeat(C):
    pb = synthetic_problem(tiny("helical_arc"), M=3)
    outs = []
    for _ in range(2):
        rec = _gpu_recon(pb)
        rec.run(5)
        outs.append(host(rec.x))
        rec.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("kind", ["axial_flat", "helical_arc", "fan2d_flat"])
def test_count_work_matches_dense_oracle_matrix(C, kind):
    """ct_count_work / ct_count_nnz (the units of the bench's algorithmic FLOP figure)
    against the oracle's dense A built column by column: nonzeros, in-cone
    voxel-view pairs and column-view pairs (float32 vs float64 footprint edges
    may flip a handful of entries)."""
    g = tiny(kind)
    shape = P.vol_shape(g)
    nv = int(np.prod(shape))
    na = g["na"]
    cols = []
    nth = P.max_threads()
    P.set_threads(1)            # ~1000 tiny calls: thread start-up would dominate
    try:
        for q in range(nv):
            e = np.zeros(nv)
            e[q] = 1.0
            cols.append(P.forward(g, e.reshape(shape)).reshape(na, -1))   # (views, rays of a view)
    finally:
        P.set_threads(nth)
    A = np.stack(cols, axis=-1) > 0                                 # (views, rays, voxels)
    nnz = int(A.sum())
    hit = A.any(axis=1)                                             # (views, voxels)
    pvox = int(hit.sum())
    pcol = int(hit.reshape(na, shape[0], -1).any(axis=1).sum())
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        a, b, c = C.ct_count_work(h, C.views(0, 1, na))
        assert a == C.ct_count_nnz(h, C.views(0, 1, na))
        assert abs(a - nnz) <= 2e-3 * nnz, (a, nnz)
        assert abs(b - pvox) <= 2e-3 * pvox, (b, pvox)
        assert abs(c - pcol) <= 2e-3 * pcol, (c, pcol)
        if g["dim"] == 2:
            assert b == c
        # additive over view subsets
        parts = [C.ct_count_work(h, C.views(m, 3, (na - m + 2) // 3)) for m in range(3)]
        assert tuple(sum(p[i] for p in parts) for i in range(3)) == (a, b, c)
    finally:
        C.ct_geom_destroy(h)


@pytest.mark.parametrize("kind,V0,M", [("fan2d_arc", 8, 3), ("axial_flat", 5, 3)])
def test_exact_subsets_gpu_M_equals_M1(C, kind, V0, M):
    """P9 on the GPU: with subsets that are exact copies of each other (M
    pitch-0 turns, tests/test_oracle_alg.py), relaxed OS-LALM with M subsets
    equals the M = 1 run sub-iteration for sub-iteration, and both match the
    oracle."""
    from tests.test_oracle_alg import repeated_turn_problem
    prob, x0 = repeated_turn_problem(kind, V0, M)
    g = prob.g
    reg = dict(potential="hyperbola", delta=0.01, betas=[5.0] * (13 if g["dim"] == 3 else 4),
               n_dirs=13 if g["dim"] == 3 else 4)
    DL = prob.D_L()
    xs = []
    for mm, iters in ((M, 2), (1, 2 * M)):
        pb = dict(geom=g, y=prob.y, w=prob.w, x0=x0, reg=reg, solver=dict(M=mm, alpha=1.999))
        rec = _gpu_recon(pb)
        rec.run(mm * iters)
        xs.append(host(rec.x))
        rec.close()
    xo, _, _ = alg.alg1(prob, x0, M, 1.999, 2, DL=DL)
    assert rel(xs[0], xs[1]) <= 1e-5, rel(xs[0], xs[1])
    assert rel(xs[0], xo) <= 1e-4, rel(xs[0], xo)


def test_sino_upload_and_host_pipeline(C):
    """ct_sino_upload copies exactly the rows of the given views; the host
    pipeline (first step subset by subset, then double-buffered whole copies)
    gives the same iterate as device-resident data (same kernels in the same
    order: bit-identical)."""
    from paper_1512_04564_b200.recon import HostPipeline
    pb = synthetic_problem(tiny("helical_arc"), M=3)
    g = pb["geom"]
    y_h = torch.as_tensor(pb["y"], dtype=torch.float32).contiguous().pin_memory()
    w_h = torch.as_tensor(pb["w"], dtype=torch.float32).contiguous().pin_memory()
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        d = torch.zeros(y_h.shape, dtype=torch.float32, device="cuda")
        C.ct_sino_upload(h, y_h, C.views(1, 3, (g["na"] - 1 + 2) // 3), d)
        want = np.zeros(y_h.shape)
        want[1::3] = y_h.double().numpy()[1::3]
        assert np.array_equal(host(d), want)
        with pytest.raises(C.CtError):
            C.ct_sino_upload(h, y_h, C.views(0, 1, g["na"] + 1), d)
    finally:
        C.ct_geom_destroy(h)
    ref = _gpu_recon(pb)
    ref.run(7)
    xr = host(ref.x)
    ref.close()
    rec = _gpu_recon(pb)
    pipe = HostPipeline(rec)
    x_h = [torch.empty(rec.x.shape, dtype=torch.float32).pin_memory() for _ in range(2)]
    pipe.enqueue_copy_in(y_h, w_h, by_subset=True)
    pipe.step(4, x_h[0], next_inputs=(y_h, w_h))
    pipe.step(3, x_h[1], next_inputs=None)
    pipe.finish()
    torch.cuda.synchronize()
    assert rec.k == 7
    assert np.array_equal(x_h[1].double().numpy(), xr)
    rec.close()


@pytest.mark.parametrize("name", ["c5", "c4", "c3", "c2"])
def test_full_size_subiteration_sampled(C, name):
    """BASELINE config at full size, bench launch configuration (graph-replayed
    solve): one sub-iteration from a seeded state (k = 5, so subset 5 and
    rho_5), compared with the oracle: x+ on every voxel; g+ and htilde+ on
    sampled voxels (the oracle back-projects the subset residual of its own
    x+ at those voxels)."""
    from oracle import alg
    from paper_1512_04564_b200.recon import Recon
    from synth.configs import get_config, reg_betas
    from synth.data import make_dataset
    cfg = get_config(name)
    g = cfg["geom"]
    M, alpha = cfg["solver"]["M"], cfg["solver"]["alpha"]
    data = make_dataset(cfg, device="cuda")
    y = data["y"].double().cpu().numpy()
    w = data["w"].double().cpu().numpy()
    x = data["x0"].double().cpu().numpy()
    shape = x.shape
    rng = np.random.default_rng(11)
    # seeded state: smooth positive D_L of the right scale, gradient-scale g and htilde
    dl = (0.5 + rng.random(shape)) * cfg["reg"]["beta0"] * 40.0
    gg = rng.standard_normal(shape) * cfg["reg"]["beta0"] * 1e-3
    ht = rng.standard_normal(shape) * cfg["reg"]["beta0"] * 1e-3
    nd = cfg["reg"]["n_dirs"]
    reg = dict(potential="hyperbola", delta=cfg["reg"]["delta"], betas=reg_betas(g, cfg["reg"]["beta0"], nd),
               n_dirs=nd)
    k0 = 5
    rec = Recon(g, reg, cfg["solver"], data["y"], data["w"], x)
    rec.set_DL(dl)
    rec.g.copy_(torch.as_tensor(gg, dtype=torch.float32))
    rec.htilde.copy_(torch.as_tensor(ht, dtype=torch.float32))
    rec.state.k = k0
    # the device state is float32: feed the oracle the same rounded inputs
    x32, g32, h32, dl32 = (np.asarray(np.float32(a), dtype=np.float64) for a in (x, gg, ht, dl))
    rec.run(1)
    xg, gg_gpu, ht_gpu = host(rec.x), host(rec.g), host(rec.htilde)
    # the solver's weighted residual of this sub-iteration (the benched forward instance, graph
    # launch) at 2048 sampled rays against the oracle's W (A x+ - y) of the GPU's own x+
    m = k0 % M
    vcount = (g["na"] - m + M - 1) // M
    nt = g["nt"] if g["dim"] == 3 else 1
    r = torch.empty((vcount, nt, g["ns"]), dtype=torch.float32, device="cuda")
    C.oslalm_residual(rec.h, rec.params, rec.k, rec.ws, r)
    rg = host(r)
    nray = 2048
    vi = rng.integers(0, vcount, nray)
    ss = rng.integers(0, g["ns"], nray)
    tt = rng.integers(0, nt, nray)
    vv = m + M * vi
    ax = P.forward_rays(g, xg, vv, ss, tt)
    wv, yv = w[vv, tt, ss], y[vv, tt, ss]
    err = np.linalg.norm(rg[vi, tt, ss] - wv * (ax - yv)) / np.linalg.norm(wv * ax)
    assert err <= 1e-4, ("residual", err)
    # both forward paths of the ABI on x0 at the same rays (all views of the subset)
    views_c = C.views(m, M, vcount)
    axo = P.forward_rays(g, x, vv, ss, tt)
    pd = torch.empty_like(r)
    C.ct_forward(rec.h, rec.x.copy_(torch.as_tensor(x, dtype=torch.float32)), views_c, pd)
    assert rel(host(pd)[vi, tt, ss], axo) <= 1e-4, ("ct_forward", rel(host(pd)[vi, tt, ss], axo))
    if g["dim"] == 3:
        wsz = torch.empty(C.ct_zprefix_size(rec.h), dtype=torch.uint8, device="cuda")
        C.ct_forward_zprefix(rec.h, rec.x, views_c, pd, wsz)
        assert rel(host(pd)[vi, tt, ss], axo) <= 1e-4, ("zprefix", rel(host(pd)[vi, tt, ss], axo))
        del wsz
    rec.close()
    # oracle, Alg. 1 lines 4-8 in the paper's variables (h = D_L x - htilde)
    prob = alg.Problem(g, y, w, reg["potential"], reg["delta"], reg["betas"], nd)
    h = dl32 * x32 - h32
    rho = alg.rho_k(k0, alpha)
    gradR, DR = prob.reg(x32)
    s = rho * (dl32 * x32 - h) + (1 - rho) * g32
    xo = np.maximum(x32 - (s + gradR) / (rho * dl32 + DR), 0.0)
    assert rel(xg, xo) <= 1e-5, rel(xg, xo)
    m = k0 % M
    views = (m, M, (g["na"] - m + M - 1) // M)
    r = w[m::M][:views[2]] * (P.forward(g, xo, views) - y[m::M][:views[2]])
    idx = np.sort(rng.choice(xo.size, 400, replace=False))
    zeta = M * P.back_voxels(g, r, views, idx)
    go = rho / (rho + 1) * (alpha * zeta + (1 - alpha) * g32.ravel()[idx]) + g32.ravel()[idx] / (rho + 1)
    ho = alpha * (dl32.ravel()[idx] * xo.ravel()[idx] - zeta) + (1 - alpha) * h.ravel()[idx]
    assert rel(gg_gpu.ravel()[idx], go) <= 1e-4, rel(gg_gpu.ravel()[idx], go)
    hto = dl32.ravel()[idx] * xo.ravel()[idx] - ho
    assert rel(ht_gpu.ravel()[idx], hto) <= 1e-4, rel(ht_gpu.ravel()[idx], hto)


@pytest.mark.parametrize("kind", ["helical_arc", "fan2d_arc"])
def test_nccl_sharded_path_world1_matches_single_gpu(C, kind):
    """The multi-GPU solve path (partial zeta -> ncclAllReduce overlapped with
    the stencil of the new x on a side stream -> fold + x-update kernel) on a
    world-1 NCCL communicator equals the fused single-GPU path, also when the
    run is split over two calls (the last zeta is folded before returning)."""
    from paper_1512_04564_b200.recon import Recon
    pb = synthetic_problem(tiny(kind), M=3)
    uid = C.ct_nccl_unique_id()
    d = C.ct_dist_create(0, 1, uid, 0)
    try:
        outs = []
        for dist, calls in ((None, (7,)), (d, (7,)), (d, (3, 4))):
            r = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], dist=dist)
            r.compute_DL()
            for n in calls:
                r.run(n)
            assert r.k == 7
            outs.append((host(r.x), host(r.g), host(r.htilde), host(r.dl)))
            r.close()
        for o in outs[1:]:
            for a, b in zip(outs[0], o):
                assert rel(b, a) <= 1e-5   # same arithmetic, different FMA contraction / order
    finally:
        C.ct_dist_destroy(d)


@pytest.mark.parametrize("kind,world", [("helical_arc", 2), ("helical_arc", 3), ("axial_flat", 2),
                                        ("helical_fine", 3), ("fan2d_arc", 1), ("helical_mid", 4)])
def test_zslab_decomposition_matches_single_gpu(C, kind, world):
    """the z-slab decomposition with `world` slabs driven by one
    process (partial projections summed on the device, halos copied) matches the
    float64 oracle (Algorithm 1 trace: D_L, and x, g, htilde after 7 sub-iterations
    split over two calls) and equals the fused single-GPU solve."""
    from paper_1512_04564_b200.recon import Recon
    from tests.geoms import mid
    pb = synthetic_problem(mid(kind) if kind.endswith("_mid") else tiny(kind), M=3)
    trace = {}
    alg.alg1(oracle_problem(pb), pb["x0"], 3, 1.999, 3, DL=pb["DL"], trace=trace)
    xo, go, ho = trace[7]
    ref = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"])
    ref.compute_DL()
    ref.run(7)
    want = [host(ref.x), host(ref.g), host(ref.htilde), host(ref.dl)]
    ref.close()
    g = pb["geom"]
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        p = C.params(3, 1.999)
        reg = C.reg_desc(pb["reg"]["potential"], pb["reg"]["delta"], pb["reg"]["betas"], pb["reg"]["n_dirs"])
        y, w = dev(pb["y"]), dev(pb["w"])
        xs, gs, hs, dls, wss, sts = [], [], [], [], [], []
        nb = max(C.oslalm_zslab_workspace_size(h, p, r, world) for r in range(world))
        for r in range(world):
            z0, nz = C.ct_zslab_range(h, r, world)
            xs.append(dev(pb["x0"][z0:z0 + nz]))
            gs.append(torch.zeros_like(xs[-1]))
            hs.append(torch.zeros_like(xs[-1]))
            dls.append(torch.empty_like(xs[-1]))
            wss.append(torch.empty(nb, dtype=torch.uint8, device="cuda"))
            sts.append(C.make_state(xs[-1], gs[-1], hs[-1], 0))
        C.ct_sqs_diag_zslab(h, w, dls, wss, world)
        assert rel(host(torch.cat(dls)), pb["DL"]) <= 1e-4
        assert rel(host(torch.cat(dls)), want[3]) <= 1e-5
        C.oslalm_zslab_solve(h, y, w, reg, dls, p, sts, 3, wss, world)
        C.oslalm_zslab_solve(h, y, w, reg, dls, p, sts, 4, wss, world)
        assert all(s_.k == 7 for s_ in sts)
        xg, gg_, hg = host(torch.cat(xs)), host(torch.cat(gs)), host(torch.cat(hs))
        assert rel(xg, xo) <= 1e-4, rel(xg, xo)
        assert rel(gg_, go) <= 1e-3
        assert rel(hg, pb["DL"] * xo - ho) <= 1e-3
        # against the fused single-GPU solve: the slabs' partial projections are summed in another
        # order (and each slab's z-prefix restarts at its bottom plane), float32 rounding only
        for name, got, exp in zip(("x", "g", "htilde"), (xg, gg_, hg), want):
            assert rel(got, exp) <= 5e-5, (name, rel(got, exp))
    finally:
        C.ct_geom_destroy(h)


def test_zslab_nccl_world1(C):
    """The z-slab driver's NCCL path (one slab per process, ncclAllReduce of the
    partial projections, halo send/recv) on a world-1 communicator."""
    pb = synthetic_problem(tiny("helical_arc"), M=3)
    from paper_1512_04564_b200.recon import Recon
    ref = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"])
    ref.compute_DL()
    ref.run(5)
    want = host(ref.x)
    ref.close()
    g = pb["geom"]
    h = C.ct_geom_create(C.geom_desc(g))
    d = C.ct_dist_create(0, 1, C.ct_nccl_unique_id(), 0)
    try:
        p = C.params(3, 1.999)
        reg = C.reg_desc(pb["reg"]["potential"], pb["reg"]["delta"], pb["reg"]["betas"], pb["reg"]["n_dirs"])
        x = dev(pb["x0"])
        gg, hh, dl = torch.zeros_like(x), torch.zeros_like(x), torch.empty_like(x)
        ws = torch.empty(C.oslalm_zslab_workspace_size(h, p, 0, 1), dtype=torch.uint8, device="cuda")
        C.ct_sqs_diag_zslab(h, dev(pb["w"]), [dl], [ws], 1, dist=d)
        st = C.make_state(x, gg, hh, 0)
        C.oslalm_zslab_solve(h, dev(pb["y"]), dev(pb["w"]), reg, [dl], p, [st], 5, [ws], 1, dist=d)
        assert rel(host(x), want) <= 1e-5
        trace = {}
        alg.alg1(oracle_problem(pb), pb["x0"], 3, 1.999, 2, DL=pb["DL"], trace=trace)
        assert rel(host(x), trace[5][0]) <= 1e-4
    finally:
        C.ct_dist_destroy(d)
        C.ct_geom_destroy(h)
