"""Convergence study on the GPU (Sec. V claims):
RMS distance to a converged reference x* per outer iteration for
  proposed relaxed OS-LALM (Alg. 1, alpha = 1.999), simple relaxed (Alg. 2,
  alpha = 1.999), unrelaxed OS-LALM (alpha = 1) with M and 2M subsets, and OS-SQS.
The reference is Alg. 1 with one subset (M = 1, the setting of the paper's
theorems) run until it stops moving.  Qualitative echoes of the paper: the
proposed method with M subsets should track the unrelaxed one with 2M subsets
("fewer subsets"), and beat the simple relaxation and OS-SQS.

usage: python scripts/convergence.py [config] [iters] [ref_iters] [--fbp]
--fbp starts every run from the FBP / FDK image of y (ct_fbp, the paper's
"initial (FBP) image"; 360-degree scans) instead of reading R17's
blurred phantom.  Writes gpurun_out/convergence_<config>[_fbp].{json,txt}; RMS
is reported in mm^-1 and in "HU" with mu_water = 0.02 mm^-1 (the synthetic
phantom's body density).
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
    fbp = "--fbp" in sys.argv
    argv = [a for a in sys.argv[1:] if a != "--fbp"]
    name = argv[0] if len(argv) > 0 else "c3"
    iters = int(argv[1]) if len(argv) > 1 else 30
    ref_iters = int(argv[2]) if len(argv) > 2 else 1500
    cfg = get_config(name)
    inp = bench.make_inputs(cfg, "cuda")
    if fbp:
        r0 = Recon(cfg["geom"], inp["reg"], cfg["solver"], inp["y"], inp["w"], inp["x0"])
        inp["x0"] = r0.init_fbp().clone().clamp_(min=0.0)   # Omega = {x >= 0}
        r0.close()
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
    out = {"config": name, "M": M, "iters": iters, "init": "FBP/FDK (ct_fbp), clamped to x >= 0" if fbp else
           "blurred voxelised phantom (DESIGN.md R17)", "ref": {"algorithm": "Alg. 1, M = 1, alpha = 1.999",
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
    lines = ["RMS(x_k - x*) in HU (mu_water = 0.02/mm), %s, M = %d, start: %s" % (name, M, out["init"]),
             "iter " + " ".join("%16s" % k for k in runs)]
    for it in list(range(0, min(iters, 10) + 1)) + list(range(15, iters + 1, 5)):
        lines.append("%4d " % it + " ".join("%16.2f" % (out["rms"][k][it] * hu) for k in runs))
    print("\n".join(lines))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = name + ("_fbp" if fbp else "")
    with open(os.path.join(ROOT, "gpurun_out", "convergence_%s.json" % tag), "w") as f:
        json.dump(out, f, indent=1)
    with open(os.path.join(ROOT, "gpurun_out", "convergence_%s.txt" % tag), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
