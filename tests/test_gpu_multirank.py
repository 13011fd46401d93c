"""View-sharded multi-GPU path on one GPU: a local
emulation of `world` ranks (ct_dist_create_local) runs rank p's share of every
subset (the device picks views p, p + world, ... from rank p's control block)
into its own partial back-projection, sums the partials in rank order (the
reduce-scatter), lets each z-slab owner fold zeta and update its slab with halo
planes from the neighbouring slabs, and rebuilds the z-prefix of the whole x+
(the all-gather).  Compared with the float64 oracle (Algorithm 1, P:333-348;
the subset gradient does not depend on how its views are split) and
with the fused single-GPU path.  Tolerances as tests/test_gpu_parity.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import alg  # noqa: E402
from tests.geoms import mid, tiny  # noqa: E402
from tests.problems import oracle_problem, rel, synthetic_problem  # noqa: E402


@pytest.fixture(scope="module")
def C():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1512_04564_b200 import ctrecon
    ctrecon.load()
    return ctrecon


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


def _geom(kind):
    return mid(kind) if kind.endswith("_mid") else tiny(kind)


CASES = [("helical_arc", 3), ("helical_arc", 2), ("axial_flat", 2), ("helical_fine", 4), ("fan2d_arc", 2),
         ("helical_mid", 3), ("helical_arc", 10)]


@pytest.mark.parametrize("kind,world", CASES)
def test_local_view_sharding_matches_oracle_and_single_gpu(C, kind, world):
    from paper_1512_04564_b200.recon import Recon
    g = _geom(kind)
    M = 3
    pb = synthetic_problem(g, M=M)
    prob = oracle_problem(pb)
    trace = {}
    alg.alg1(prob, pb["x0"], M, 1.999, 2, DL=pb["DL"], trace=trace)
    ref = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"])
    ref.compute_DL()
    ref.run(2 * M)
    want = [host(ref.x), host(ref.g), host(ref.htilde), host(ref.dl)]
    ref.close()
    d = C.ct_dist_create_local(world, 0)
    try:
        rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], dist=d)
        rec.compute_DL()
        assert rel(host(rec.dl), pb["DL"]) <= 1e-4
        assert rel(host(rec.dl), want[3]) <= 1e-5
        done = 0
        for k in (1, 2, 4, 2 * M):          # one call each: resumes across calls
            rec.run(k - done)
            done = k
            xo, go, ho = trace[k]
            assert rec.k == k
            assert rel(host(rec.x), xo) <= 1e-4, (k, rel(host(rec.x), xo))
            assert rel(host(rec.g), go) <= 1e-3, (k, rel(host(rec.g), go))
            assert rel(host(rec.htilde), pb["DL"] * xo - ho) <= 1e-3, k
        # CUDA against CUDA (the oracle checks above are the parity bar): the same arithmetic with
        # zeta's partial sums in another order; g and htilde accumulate alpha zeta in float32 at
        # magnitudes ~4e3 (differences of the order of 1e-5 relative are rounding, e.g. 1.5e-5 on
        # helical_mid with 3 shards), x stays within 1e-5
        for a, b, tol in zip((host(rec.x), host(rec.g), host(rec.htilde)), want[:3], (1e-5, 5e-5, 5e-5)):
            assert rel(a, b) <= tol, rel(a, b)
        # the residual of rank 0's share of the last sub-iteration against the oracle
        m = (2 * M - 1) % M
        vm = (g["na"] - m + M - 1) // M
        cnt = (vm + world - 1) // world
        views = (m, M * world, cnt)
        nt = g["nt"] if g["dim"] == 3 else 1
        r = torch.empty((cnt, nt, g["ns"]), dtype=torch.float32, device="cuda")
        C.oslalm_residual(rec.h, rec.params, rec.k, rec.ws, r, dist=d)
        from oracle import projector as P
        xk = trace[2 * M][0]
        ax = P.forward(g, xk, views)
        wv = pb["w"][m::M * world][:cnt]
        ro = wv * (ax - pb["y"][m::M * world][:cnt])
        assert np.linalg.norm(host(r) - ro) <= 1e-4 * np.linalg.norm(wv * ax)
        rec.close()
    finally:
        C.ct_dist_destroy(d)


def test_local_view_sharding_kappa_and_alg2(C):
    """kappa weights through the slab stencil's halo planes, and Algorithm 2, on 3 emulated ranks."""
    from paper_1512_04564_b200.recon import Recon
    g = tiny("helical_arc")
    pb = synthetic_problem(g, M=3)
    rng = np.random.default_rng(5)
    kap = rng.uniform(0.6, 1.4, pb["x0"].shape)
    prob = oracle_problem(pb)
    prob.kappa = kap
    xo = alg.alg1(prob, pb["x0"], 3, 1.999, 2, DL=pb["DL"])[0]
    d = C.ct_dist_create_local(3, 0)
    try:
        rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], kappa=kap, dist=d)
        rec.set_DL(pb["DL"])
        rec.run(6)
        assert rel(host(rec.x), xo) <= 1e-4
        rec.close()
        prob.kappa = None
        xs, gs = alg.alg2(prob, pb["x0"], 3, 1.999, 2, DL=pb["DL"])
        rec = Recon(pb["geom"], pb["reg"], dict(pb["solver"], variant="simple"), pb["y"], pb["w"], pb["x0"], dist=d)
        rec.set_DL(pb["DL"])
        rec.run(4)
        rec.run(2)
        assert rel(host(rec.x), xs) <= 1e-4
        assert rel(host(rec.g), gs) <= 1e-3
        rec.close()
    finally:
        C.ct_dist_destroy(d)


def test_local_world_larger_than_planes_is_rejected(C):
    from paper_1512_04564_b200.recon import Recon
    pb = synthetic_problem(tiny("helical_arc"), M=3)   # nz = 10
    d = C.ct_dist_create_local(11, 0)
    try:
        rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], dist=d)
        rec.set_DL(pb["DL"])
        x0 = rec.x.clone()
        with pytest.raises(C.CtError) as e:
            rec.run(1)
        assert e.value.status == C.CT_E_CONFIG and rec.k == 0 and torch.equal(rec.x, x0)
        rec.close()
    finally:
        C.ct_dist_destroy(d)


@pytest.mark.parametrize("kind,world,nseg", [("helical_mid", 2, 3), ("helical_mid", 4, 2)])
def test_local_view_sharding_segmented_forward(C, kind, world, nseg):
    """The emulated ranks with the segmented forward (ct_geom_set_fwd_segments, automatic at
    c5): every rank's forward runs through its own schedule key (view stride world * M) and
    the shared partial buffer; x, g, htilde against the oracle after 1, 3 and 2M sub-iterations."""
    from paper_1512_04564_b200.recon import Recon
    g = _geom(kind)
    M = 3
    pb = synthetic_problem(g, M=M)
    prob = oracle_problem(pb)
    trace = {}
    alg.alg1(prob, pb["x0"], M, 1.999, 2, DL=pb["DL"], trace=trace)
    d = C.ct_dist_create_local(world, 0)
    try:
        rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], dist=d, fwd_segments=nseg)
        assert C.ct_geom_fwd_segments(rec.h, 200) == nseg
        rec.set_DL(pb["DL"])
        done = 0
        for k in (1, 3, 2 * M):
            rec.run(k - done)
            done = k
            xo, go, ho = trace[k]
            assert rel(host(rec.x), xo) <= 1e-4, (k, rel(host(rec.x), xo))
            assert rel(host(rec.g), go) <= 1e-3, (k, rel(host(rec.g), go))
            assert rel(host(rec.htilde), pb["DL"] * xo - ho) <= 1e-3, k
        rec.close()
    finally:
        C.ct_dist_destroy(d)
