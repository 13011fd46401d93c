"""Convergence study on the GPU (Sec. V claims):
RMS distance to a converged reference x* per outer iteration for
  proposed relaxed OS-LALM (Alg. 1, alpha = 1.999), simple relaxed (Alg. 2,
  alpha = 1.999), unrelaxed OS-LALM (alpha = 1) with M and 2M subsets, and OS-SQS.
The reference is Alg. 1 with one subset (M = 1, the setting of the paper's
theorems) run until it stops moving.  Qualitative echoes of the paper: the
proposed method with M subsets should track the unrelaxed one with 2M subsets
("fewer subsets"), and beat the simple relaxation and OS-SQS.

usage: python scripts/convergence.py [config] [iters] [ref_iters]
Writes profiles/convergence_<config>.json; RMS is reported in mm^-1 and in
"HU" with mu_water = 0.02 mm^-1 (the synthetic phantom's body density).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1512_04564_b200.recon import Recon  # noqa: E402
from synth.configs import get_config  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    ref_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
    cfg = get_config(name)
    inp = bench.make_inputs(cfg, "cuda")
    g = cfg["geom"]
    M = cfg["solver"]["M"]
    base = dict(cfg["solver"])

    def recon(**solver):
        s = dict(base)
        reg = dict(inp["reg"])
        reg.update(solver.pop("reg", {}))
        solver.pop("dl_scale", None)
        s.update(solver)
        r = Recon(g, reg, s, inp["y"], inp["w"], inp["x0"])
        return r

    # reference: Alg. 1, M = 1, alpha = 1.999, until converged
    t0 = time.time()
    ref = recon(M=1, alpha=1.999)
    ref.compute_DL()
    dl = ref.dl.clone()
    prev = ref.x.clone()
    moves = []
    for blk in range(ref_iters // 100):
        ref.run(100)
        torch.cuda.synchronize()
        mv = float((ref.x - prev).norm() / ref.x.norm())
        moves.append(mv)
        prev = ref.x.clone()
    xref = ref.x.clone()
    t_ref = time.time() - t0
    runs = {
        "proposed_M": dict(M=M, alpha=1.999),
        "simple_M": dict(M=M, alpha=1.999, variant="simple"),
        "unrelaxed_M": dict(M=M, alpha=1.0),
        "unrelaxed_2M": dict(M=2 * M, alpha=1.0),
        "os_sqs_M": dict(M=M, alpha=1.0, variant="simple", rho_mode="fixed", rho_fixed=1.0),
        # supplement P:1272: majorization study (maximum vs Huber curvature; D_L scaled by 2)
        "proposed_maxcurv": dict(M=M, alpha=1.999, reg=dict(curvature="max")),
        "proposed_2DL": dict(M=M, alpha=1.999, dl_scale=2.0),
    }
    out = {"config": name, "M": M, "iters": iters, "ref": {"algorithm": "Alg. 1, M = 1, alpha = 1.999",
           "iters": ref_iters, "rel_move_per_100_iters": moves, "seconds": t_ref}, "rms": {}}
    x0_rms = float((inp["x0"].to(xref.device) - xref).pow(2).mean().sqrt())
    for key, sv in runs.items():
        r = recon(**dict(sv))
        r.set_DL(dl * sv.get("dl_scale", 1.0))   # study harness: D_L majorizer scaled
        rms = [x0_rms]
        for it in range(iters):
            r.run(sv["M"])
            rms.append(float((r.x - xref).pow(2).mean().sqrt()))
        out["rms"][key] = rms
        r.close()
    ref.close()
    hu = 1000.0 / 0.02
    lines = ["RMS(x_k - x*) in HU (mu_water = 0.02/mm), %s, M = %d" % (name, M),
             "iter " + " ".join("%16s" % k for k in runs)]
    for it in list(range(0, min(iters, 10) + 1)) + list(range(15, iters + 1, 5)):
        lines.append("%4d " % it + " ".join("%16.2f" % (out["rms"][k][it] * hu) for k in runs))
    print("\n".join(lines))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "convergence_%s.json" % name), "w") as f:
        json.dump(out, f, indent=1)
    with open(os.path.join(ROOT, "gpurun_out", "convergence_%s.txt" % name), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
