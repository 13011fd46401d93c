"""A small workload that launches every kernel family of libctrecon.so, for
compute-sanitizer (racecheck / synccheck / memcheck):

  * 3-D solve on the mid-size helical geometry (the forward's warp queue, the
    cp.async y/w staging, the update's per-row named barriers and z-prefix
    exchange, the back-projector's shared row buffers and view-descriptor
    staging), flat RPL = 4 and axial geometries, graph-replayed;
  * ct_forward / ct_forward_zprefix / ct_back / ct_sqs_diag / ct_reg_grad /
    ct_kappa_weights / ct_fbp;
  * the emulated 3-rank view-sharded path (slab updates with halos, side stream);
  * a cropped c3 (axial cone, 64^2 x 16 of the 256^2 x 64 config) and c1 (2-D).

usage: python scripts/sanitize_run.py [--quick]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1512_04564_b200 import ctrecon as C  # noqa: E402
from paper_1512_04564_b200.recon import Recon  # noqa: E402
from synth.configs import get_config, reg_betas, shrink  # noqa: E402
from tests.geoms import mid, tiny  # noqa: E402


def problem(g, M=2, seed=0):
    rng = np.random.default_rng(seed)
    shape = (g["nz"] if g["dim"] == 3 else 1, g["ny"], g["nx"])
    nt = g["nt"] if g["dim"] == 3 else 1
    x0 = 0.02 * rng.random(shape)
    y = rng.random((g["na"], nt, g["ns"]))
    w = 1.0 + rng.random((g["na"], nt, g["ns"]))
    nd = 13 if g["dim"] == 3 else 4
    reg = dict(potential="hyperbola", delta=0.01, betas=[50.0] * nd, n_dirs=nd)
    return dict(geom=g, y=y, w=w, x0=x0, reg=reg, solver=dict(M=M, alpha=1.999))


def run_solve(pb, n=3, dist=None, kappa=None):
    rec = Recon(pb["geom"], pb["reg"], pb["solver"], pb["y"], pb["w"], pb["x0"], dist=dist, kappa=kappa)
    rec.compute_DL()
    rec.run(n)
    rec.run(1)
    torch.cuda.synchronize()
    rec.close()


def run_ops(g):
    h = C.ct_geom_create(C.geom_desc(g))
    try:
        nt = g["nt"] if g["dim"] == 3 else 1
        shape = (g["nz"] if g["dim"] == 3 else 1, g["ny"], g["nx"])
        x = torch.rand(shape, device="cuda")
        p = torch.empty((g["na"], nt, g["ns"]), device="cuda")
        v = C.views(0, 1, g["na"])
        C.ct_forward(h, x, v, p)
        ws = torch.empty(max(C.ct_zprefix_size(h), 16), dtype=torch.uint8, device="cuda")
        C.ct_forward_zprefix(h, x, v, p, ws)
        b = torch.empty_like(x)
        C.ct_back(h, p, v, b)
        C.ct_back(h, p, C.views(1, 2, (g["na"] - 1) // 2), b, scale=0.5, accumulate=True)
        d = torch.empty_like(x)
        ws2 = torch.empty(5 * g["ns"] * nt * 4, dtype=torch.uint8, device="cuda")
        C.ct_sqs_diag(h, torch.ones_like(p), d, ws2)
        nd = 13 if g["dim"] == 3 else 4
        gr, cv = torch.empty_like(x), torch.empty_like(x)
        C.ct_reg_grad(h, C.reg_desc("hyperbola", 0.01, [1.0] * nd, nd), x, gr, cv)
        C.ct_reg_grad(h, C.reg_desc("fair", 0.01, [1.0] * nd, nd), x, gr, cv, kappa=torch.rand_like(x) + 0.5)
        ws3 = torch.empty(x.numel() * 4 + 256 + 4 * g["ns"] * nt * 4, dtype=torch.uint8, device="cuda")
        C.ct_kappa_weights(h, p, d, ws3)
        if g["orbit_deg"] == 360.0 and (g["dim"] == 2 or g["pitch"] == 0.0):
            ws4 = torch.empty(p.numel() * 4, dtype=torch.uint8, device="cuda")
            C.ct_fbp(h, p, d, ws4)
        torch.cuda.synchronize()
    finally:
        C.ct_geom_destroy(h)


def main():
    quick = "--quick" in sys.argv
    C.load()
    geoms = [mid("helical_mid", na=240), mid("helical_rpl4", na=120), mid("axial_mid", na=60), tiny("fan2d_arc")]
    for g in geoms:
        run_ops(g)
        run_solve(problem(g))
        print("ok", g["dim"], g["nx"], g["ny"], g["nz"], g["ns"], g["nt"], g["na"], flush=True)
    d = C.ct_dist_create_local(3, 0)
    try:
        pb = problem(mid("helical_mid", na=120))
        run_solve(pb, n=3, dist=d, kappa=np.ones(pb["x0"].shape) * 1.1)
    finally:
        C.ct_dist_destroy(d)
    print("ok dist-local", flush=True)
    if not quick:
        for name, kw in (("c3", dict(nx=64, nz=16, na=123)), ("c1", {})):
            cfg = get_config(name)
            if kw:
                cfg = shrink(cfg, **kw)
            g = cfg["geom"]
            pb = problem(g, M=cfg["solver"]["M"] // 3 if name == "c3" else cfg["solver"]["M"])
            nd = cfg["reg"]["n_dirs"]
            pb["reg"]["betas"] = reg_betas(g, 1e3, nd)
            run_ops(g)
            run_solve(pb, n=2)
            print("ok", name, flush=True)
    print("SANITIZE_RUN_DONE")


if __name__ == "__main__":
    main()
