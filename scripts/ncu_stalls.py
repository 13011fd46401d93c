"""Stall-sample attribution of an `ncu --set full --import-source on` capture:
per kernel, the instructions whose share of the warp-stall samples most
exceeds their share of the executed instructions (the dependency chains that
wait on memory), and the stall / instruction shares by opcode.

usage: python scripts/ncu_stalls.py <prof.ncu-rep> [kernel-regex ...] [--top N]
(the source page is read with `ncu -i ... --page source --csv --print-source sass`)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def source_rows(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kernel,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h = rows[1]
    ia, isrc = h.index("Address"), h.index("Source")
    ie, ist = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    res = []
    for r in rows[2:]:
        # several kernels match the regex: each adds its own header / blank rows -- skip those
        if len(r) <= max(ia, isrc, ie, ist):
            continue
        try:
            int(r[ia], 16)
        except ValueError:
            continue
        e = int(r[ie]) if r[ie].isdigit() else 0
        s = int(r[ist]) if r[ist].isdigit() else 0
        res.append((int(r[ia], 16) & 0xffff, e, s, r[isrc].strip()))
    return list(dict.fromkeys(res))   # a kernel listed twice on the page: count each row once


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    top = 10
    if "--top" in sys.argv:
        top = int(sys.argv[sys.argv.index("--top") + 1])
        args = [a for a in args if a != str(top)]
    rep, kernels = args[0], args[1:] or ["k_fwd3", "k_back3", "k_update"]
    for k in kernels:
        rows = source_rows(rep, k)
        if not rows:
            print("== %s: no source rows" % k)
            continue
        te = sum(r[1] for r in rows) or 1
        ts = sum(r[2] for r in rows) or 1
        print("== %s  (%d instructions, %d stall samples)" % (k, te, ts))
        for a, e, s, src in sorted(rows, key=lambda r: -(r[2] / ts - r[1] / te))[:top]:
            print("  0x%04x  inst %6.3f%%  stall %6.2f%%  %s" % (a, 100 * e / te, 100 * s / ts, src[:64]))
        byop = defaultdict(lambda: [0, 0])
        for a, e, s, src in rows:
            toks = src.split()
            if not toks:
                continue
            op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
            byop[op][0] += e
            byop[op][1] += s
        print("  by opcode (stall share, instruction share):")
        for op, (e, s) in sorted(byop.items(), key=lambda x: -x[1][1])[:8]:
            print("    %-8s stall %5.1f%%  inst %5.1f%%" % (op, 100 * s / ts, 100 * e / te))


if __name__ == "__main__":
    main()
