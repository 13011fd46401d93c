"""Oracle-only reference images for the full-size parity tests (tests/golden/).

The north star's Target (BASELINE.json) is "relaxed OS-LALM on the 3-D helical
config matches the oracle ... images within 1e-3 relative RMS after a fixed
number of iterations".  The float64 oracle needs ~25 min per config on 8
cores, longer than the GPU test step may take, so this script runs it once,
here, and stores what the GPU tests compare against.  It calls only oracle/
(Algorithm 1, and the SF projector) and the seeded input
generators (synth/, via tests/problems.py); nothing comes from the CUDA path.

    python scripts/oracle_golden.py c2   # 30 outer iterations (BASELINE configs[1], 2-D); full image
    python scripts/oracle_golden.py c3   # 30 outer iterations (BASELINE configs[2]); full image
    python scripts/oracle_golden.py c4   # 1 outer iteration = 24 sub-iterations (configs[3]); sampled

Stored (tests/golden/<cfg>_alg1.npz):
  x        x after the run: the whole volume (float32) for c3; for c4 the
           values at NSAMP voxels drawn by np.random.default_rng(SEED)
           (float64; the 96 MiB volume is not committed)
  idx      flat voxel indices of the samples (c4)
  dl       D_L = diag(A'WA1) at the same voxels (c4; c3: sampled too)
  fp_*     fingerprints of the inputs (y, w, x0): the GPU test regenerates them
           with synth/ on the host and checks they are the same arrays
  subiters, seconds, threads
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import alg  # noqa: E402
from oracle import projector as P  # noqa: E402
from tests.problems import config_problem, input_fingerprint, oracle_problem  # noqa: E402

SEED = 20240
NSAMP = 1 << 18
OUTER = {"c2": 30, "c3": 30, "c4": 1}


def main(name):
    t0 = time.perf_counter()
    pb = config_problem(name)          # synth inputs on the host + oracle D_L (all views)
    t_dl = time.perf_counter() - t0
    prob = oracle_problem(pb)
    M, alpha = pb["solver"]["M"], pb["solver"]["alpha"]
    iters = OUTER[name]
    t1 = time.perf_counter()
    x, g, h = alg.alg1(prob, pb["x0"], M, alpha, iters, DL=pb["DL"])
    t_run = time.perf_counter() - t1
    rng = np.random.default_rng(SEED)
    idx = np.sort(rng.choice(x.size, min(NSAMP, x.size), replace=False))
    out = dict(idx=idx, dl=pb["DL"].ravel()[idx], subiters=M * iters, threads=P.max_threads(),
               seconds=np.array([t_dl, t_run]))
    if name in ("c2", "c3"):
        out["x"] = x.astype(np.float32)
    else:
        out["x"] = x.ravel()[idx]
    out.update({"fp_" + k: v for k, v in input_fingerprint(pb).items()})
    path = os.path.join(ROOT, "tests", "golden", "%s_alg1.npz" % name)
    np.savez_compressed(path, **out)
    print(json.dumps({"config": name, "subiters": M * iters, "data_and_DL_s": t_dl, "alg1_s": t_run,
                      "threads": P.max_threads(), "path": path, "bytes": os.path.getsize(path)}))


if __name__ == "__main__":
    for n in sys.argv[1:]:
        main(n)
