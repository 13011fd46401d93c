"""Seeded test problems shared by CPU and GPU tests (inputs only + oracle refs)."""
import numpy as np

from oracle import alg
from oracle import projector as P
from synth.configs import get_config, reg_betas
from synth.data import make_dataset


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def beta0_from_DL(DL, geom, n_dirs, c_beta=0.05):
    """beta0 = c * median_{D_L>0}(D_L) / (4 sum_i w_i)."""
    w = reg_betas(geom, 1.0, n_dirs)
    pos = DL[DL > 0]
    return c_beta * float(np.median(pos)) / (4.0 * sum(w))


def synthetic_problem(geom, seed=0, I0=1e4, n_dirs=None, potential="hyperbola", delta=0.01, M=4, alpha=1.999):
    """Random smooth phantom on an arbitrary (small) geometry; oracle D_L and betas."""
    rng = np.random.default_rng(seed)
    shape = P.vol_shape(geom)
    nz, ny, nx = shape
    zz, yy, xx = np.meshgrid(np.linspace(-1, 1, nz), np.linspace(-1, 1, ny), np.linspace(-1, 1, nx), indexing="ij")
    xt = 0.02 * ((xx ** 2 + yy ** 2 + 0.5 * zz ** 2) < 0.7) + 0.005 * rng.random(shape)
    ell = P.forward(geom, xt)
    c = np.maximum(rng.poisson(I0 * np.exp(-ell)).astype(np.float64), 1.0)
    y = np.log(I0 / c)
    w = c
    if n_dirs is None:
        n_dirs = 13 if geom["dim"] == 3 else 4
    DL = P.back(geom, w * P.forward(geom, np.ones(shape)))
    b0 = beta0_from_DL(DL, geom, n_dirs)
    betas = reg_betas(geom, b0, n_dirs)
    x0 = np.clip(xt + 0.003 * rng.standard_normal(shape), 0, None)
    return dict(geom=geom, y=y, w=w, x0=x0, xt=xt, DL=DL,
                reg=dict(potential=potential, delta=delta, betas=betas, n_dirs=n_dirs),
                solver=dict(M=M, alpha=alpha))


def input_fingerprint(pb):
    """Fingerprints of a problem's inputs (y, w, x0): element count, sum and sum of
    squares (float64) — a regenerated input set must reproduce them."""
    out = {}
    for k in ("y", "w", "x0"):
        a = np.asarray(pb[k], dtype=np.float64)
        out[k] = np.array([a.size, float(a.sum()), float((a * a).sum())])
    return out


def config_problem(name, device="cpu", with_DL=True, **shrink):
    """A BASELINE config's seeded inputs (synth) with oracle D_L (with_DL) and betas."""
    from synth.configs import shrink as shrink_cfg
    cfg = get_config(name)
    if shrink:
        cfg = shrink_cfg(cfg, **shrink)
    g = cfg["geom"]
    data = make_dataset(cfg, device=device)
    y = data["y"].cpu().numpy()
    w = data["w"].cpu().numpy()
    x0 = data["x0"].cpu().numpy()
    if not with_DL and cfg["reg"]["beta0"] is None:
        raise ValueError("with_DL=False needs a calibrated beta0")
    DL = P.back(g, w * P.forward(g, np.ones(P.vol_shape(g)))) if with_DL else None
    n_dirs = cfg["reg"]["n_dirs"]
    b0 = cfg["reg"]["beta0"] if cfg["reg"]["beta0"] is not None else beta0_from_DL(DL, g, n_dirs)
    betas = reg_betas(g, b0, n_dirs)
    return dict(geom=g, y=y, w=w, x0=x0, xt=data["x_true"].cpu().numpy(), DL=DL,
                reg=dict(potential=cfg["reg"]["potential"], delta=cfg["reg"]["delta"], betas=betas,
                         n_dirs=n_dirs),
                solver=dict(cfg["solver"]))


def oracle_problem(pb):
    r = pb["reg"]
    return alg.Problem(pb["geom"], pb["y"], pb["w"], r["potential"], r["delta"], r["betas"], r["n_dirs"],
                       q=r.get("q", 1.2), curvature=r.get("curvature", "huber"))
