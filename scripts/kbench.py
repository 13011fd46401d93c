"""Per-kernel device times of one outer iteration (oslalm_profile) for a config.
usage: python scripts/kbench.py [config] [reps] [--lib variants/name.so] [--nseg N]
(--lib: a tuning variant of the library; --nseg: ct_geom_set_fwd_segments, default automatic)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1512_04564_b200 import ctrecon as C  # noqa: E402
from paper_1512_04564_b200.recon import Recon  # noqa: E402
from synth.configs import get_config  # noqa: E402

args = [a for a in sys.argv[1:]]
lib = None
if "--lib" in args:
    i = args.index("--lib")
    lib = args[i + 1]
    del args[i:i + 2]
    C.LIB_PATH = os.path.abspath(lib)
nseg = None
if "--nseg" in args:
    i = args.index("--nseg")
    nseg = int(args[i + 1])
    del args[i:i + 2]
cfg = get_config(args[0] if len(args) > 0 else "c4")
reps = int(args[1]) if len(args) > 1 else 2
inp = bench.make_inputs(cfg, "cuda")
rec = Recon(cfg["geom"], inp["reg"], cfg["solver"], inp["y"], inp["w"], inp["x0"], fwd_segments=nseg)
rec.compute_DL()
M = cfg["solver"]["M"]
rec.run(M)
for r in range(reps):
    kms = C.oslalm_profile(rec.h, rec.y, rec.w, rec.reg, rec.kappa, rec.dl, rec.params, rec.state, M, rec.ws)
    print("lib=%s nseg=%d update %.4f fwd %.4f back %.4f ms/subiter" % (
        os.path.basename(C.LIB_PATH), C.ct_geom_fwd_segments(rec.h, (cfg["geom"]["na"] + M - 1) // M),
        kms[0] / M, kms[1] / M, kms[2] / M))
