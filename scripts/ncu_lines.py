"""Executed warp instructions of one kernel per CUDA source line (ncu source page, cuda,sass view)
from a capture with `--section SourceCounters --import-source on`, largest first, with the
share of the kernel's total and of the stall samples — where a kernel's instructions go.

usage: python scripts/ncu_lines.py <prof.ncu-rep> [kernel-regex] [--top N]
"""
import csv
import io
import os
import subprocess
import sys


def main():
    args = sys.argv[1:]
    top = 45
    if "--top" in args:
        i = args.index("--top")
        top = int(args[i + 1])
        del args[i:i + 2]
    rep = args[0]
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if len(args) > 1:
        cmd += ["--kernel-name", "regex:" + args[1]]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = "?"
    hdr = None
    lines = []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            ist = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or not r or r[0] == "" or len(r) < len(hdr):
            continue
        n = int(r[ie]) if r[ie].isdigit() else 0
        s = int(r[ist]) if r[ist].isdigit() else 0
        lines.append((n, s, fname, r[0], r[1]))
    tot = sum(x[0] for x in lines)
    tst = sum(x[1] for x in lines)
    print("total %d warp instructions, %d stall samples" % (tot, tst))
    for n, s, f, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
        print("%6.2f%% inst %6.2f%% stall  %-16s L%-4s %s" % (100.0 * n / max(tot, 1), 100.0 * s / max(tst, 1), f, ln,
                                                             src.strip()[:100]))


if __name__ == "__main__":
    main()
