"""Choose beta0 per config with the ORACLE only:
    beta0 = 0.05 * median_{D_L > 0}(D_L) / (4 * sum_i w_i),  D_L = A'WA1.
For c4/c5 D_L is estimated from every q-th view (scaled by q): beta0 is a
calibration constant, not a parity value.  Prints a dict for synth/configs.py.
Run: python scripts/calibrate_beta.py c1 c2 c3 c4 c5
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import projector as P  # noqa: E402
from synth.configs import get_config, reg_betas  # noqa: E402
from synth.phantom import analytic_sinogram, sample_ellipsoids  # noqa: E402

STEP = {"c1": 1, "c2": 1, "c3": 1, "c4": 8, "c5": 41}


def main(names):
    out = {}
    for name in names:
        cfg = get_config(name)
        g = cfg["geom"]
        q = STEP[name]
        views = torch.arange(0, g["na"], q, dtype=torch.float64)
        ells = sample_ellipsoids(g, cfg["phantom"]["n_ellipsoids"], cfg["phantom"]["seed"])
        ell = analytic_sinogram(g, ells, views=views, sub_s=1, sub_t=1).numpy()
        rng = np.random.default_rng(cfg["noise"]["seed"])
        I0 = cfg["noise"]["I0"]
        c = rng.poisson(I0 * np.exp(-ell)).astype(np.float64)
        if cfg["noise"]["sigma"] > 0:
            c += cfg["noise"]["sigma"] * rng.standard_normal(c.shape)
        w = np.maximum(c, 1.0)
        vd = (0, q, views.numel())
        DL = q * P.back(g, w * P.forward(g, np.ones(P.vol_shape(g)), vd), vd)
        nd = cfg["reg"]["n_dirs"]
        b0 = 0.05 * float(np.median(DL[DL > 0])) / (4.0 * sum(reg_betas(g, 1.0, nd)))
        out[name] = float("%.4g" % b0)
        print(name, out[name], flush=True)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3"])
