"""Timing of the z-slab decomposition driven by one process on one GPU
(SURVEY.md 8f row f1).  With `world` slabs run back to back on the same
device the total device time is the sum of the per-slab work plus the
partial-projection sum; dividing by `world` estimates the per-GPU compute of a
`world`-GPU run (the NCCL all-reduce of 4 V_m nt ns bytes and the halo planes
come on top).  usage: python scripts/zslab_bench.py [config] [world ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1512_04564_b200 import ctrecon as C  # noqa: E402
from synth.configs import get_config  # noqa: E402


def main():
    args = sys.argv[1:]
    if "--lib" in args:   # a tuning variant of the library (scripts/build_variants.py)
        i = args.index("--lib")
        C.LIB_PATH = os.path.abspath(args[i + 1])
        del args[i:i + 2]
    name = args[0] if len(args) > 0 else "c4"
    worlds = [int(a) for a in args[1:]] or [1, 2, 4, 8]
    cfg = get_config(name)
    inp = bench.make_inputs(cfg, "cuda")
    g = cfg["geom"]
    M, alpha = cfg["solver"]["M"], cfg["solver"]["alpha"]
    h = C.ct_geom_create(C.geom_desc(g))
    p = C.params(M, alpha)
    r = inp["reg"]
    reg = C.reg_desc(r["potential"], r["delta"], r["betas"], r["n_dirs"])
    y, w = inp["y"], inp["w"]
    for world in worlds:
        xs, sts, dls, wss = [], [], [], []
        nb = max(C.oslalm_zslab_workspace_size(h, p, k, world) for k in range(world))
        keep = []
        for k in range(world):
            z0, nz = C.ct_zslab_range(h, k, world)
            x = inp["x0"][z0:z0 + nz].contiguous().clone()
            gg, hh, dl = torch.zeros_like(x), torch.zeros_like(x), torch.empty_like(x)
            keep += [x, gg, hh]
            xs.append(x)
            dls.append(dl)
            wss.append(torch.empty(nb, dtype=torch.uint8, device="cuda"))
            sts.append(C.make_state(x, gg, hh, 0))
        C.ct_sqs_diag_zslab(h, w, dls, wss, world)
        C.oslalm_zslab_solve(h, y, w, reg, dls, p, sts, M, wss, world)   # warm-up incl. line 1
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        C.oslalm_zslab_solve(h, y, w, reg, dls, p, sts, M, wss, world)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / M
        print("%s world=%d: %.3f ms per sub-iteration for all slabs on one GPU, %.3f ms per slab "
              "(partial sinogram %.1f MB per sub-iteration)" % (
                  name, world, ms, ms / world, 4.0 * ((g["na"] + M - 1) // M) * g["nt"] * g["ns"] / 1e6))
    C.ct_geom_destroy(h)


if __name__ == "__main__":
    main()
