"""Summarise an ncu launch list + an ncu --set full capture into profiles/<tag>/.

usage: python scripts/ncu_summary.py <tag> <launches.csv> <prof.ncu-rep> [bench.log] [config]
Writes profiles/<tag>/summary.md, kernels.csv (per-kernel launch times) and
profiles/traffic_<config>.json (DRAM bytes per launch of the three hot kernels,
read by bench.py's roofline.traffic; config defaults to c4).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    m = re.match(r"(?:void )?(?:ctr::)?(\w+)(<[^(]*>)?", name)
    base = m.group(1) if m else name[:40]
    tmpl = (m.group(2) or "") if m else ""
    return base + tmpl.replace("(bool)", "").replace("(int)", "").replace(" ", "")


def launch_table(path):
    rows = []
    with open(path) as f:
        txt = f.read()
    start = txt.find('"ID"')
    rd = csv.DictReader(io.StringIO(txt[start:]))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        rows.append((short(r["Kernel Name"]), ns))
    return rows


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append(d)
    return res


def main():
    tag, lpath, rep = sys.argv[1:4]
    blog = sys.argv[4] if len(sys.argv) > 4 and sys.argv[4] != "-" else None
    cfg = sys.argv[5] if len(sys.argv) > 5 else "c4"
    od = os.path.join(ROOT, "profiles", tag)
    os.makedirs(od, exist_ok=True)
    lt = launch_table(lpath)
    agg = defaultdict(lambda: [0, 0.0])
    for n, ns in lt:
        agg[n][0] += 1
        agg[n][1] += ns
    with open(os.path.join(od, "kernels.csv"), "w") as f:
        f.write("kernel,launches,total_us,avg_us\n")
        for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write("%s,%d,%.1f,%.2f\n" % (n, c, t / 1e3, t / 1e3 / c))
    # the sub-iteration kernels of the solve (graph replays + profiled eager run)
    # the solve's sub-iteration kernels: update, forward with the residual epilogue (MODE 1), back with
    # the g/htilde epilogue (EPI 3), advance
    sub = {k: v for k, v in agg.items() if k.startswith(("k_update<", "k_advance")) or
           re.fullmatch(r"k_fwd3<\d,[01],\d,1(?:,\d)*>|k_fwd3_reduce<\d,1>|k_fwd2<\d,1>|k_back3<\d,3,0,\d+>|k_back2<\d,3,\d>", k)}
    tot = sum(v[1] for v in sub.values())
    lines = ["# ncu summary %s" % tag, "",
             "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of "
             "`python bench.py --config %s --steps 1 --warmup 1 --no-e2e --no-cpu-baseline`.  Times are "
             "cold-cache and serialised: compare shares, not absolutes." % cfg, "",
             "| sub-iteration kernel | launches | avg us | share of sub-iteration |", "|---|---|---|---|"]
    for n, (c, t) in sorted(sub.items(), key=lambda kv: -kv[1][1]):
        lines.append("| `%s` | %d | %.1f | %.1f%% |" % (n, c, t / 1e3 / c, 100 * t / tot))
    metrics = raw_metrics(rep)
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__inst_executed.sum"]
    urow = dict(zip(list(csv.reader(io.StringIO(subprocess.run(
        ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))[0],
        list(csv.reader(io.StringIO(subprocess.run(
            ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))[1]))
    lines += ["", "Full capture (`ncu --set full --clock-control none`), one launch per kernel "
              "(units: " + ", ".join("%s [%s]" % (w, urow.get(w, "")) for w in want[:3]) + "):", "",
              "| kernel | " + " | ".join(w.split(".")[0].replace("__", ".") + ("" if "pct" not in w else " %")
                                       for w in want) + " |",
              "|---" * (len(want) + 1) + "|"]
    traffic, inst = {}, {}
    for d in metrics:
        n = short(d.get("Kernel Name", ""))
        vals = []
        for w in want:
            v = d.get(w, "")
            vals.append(v)
        lines.append("| `%s` | " % n + " | ".join(vals) + " |")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            unit = metrics[0].get("dram__bytes_read.sum", "")
        except Exception:
            continue
        key = "forward" if n.startswith(("k_fwd3", "k_fwd2")) else "back" if n.startswith("k_back") else \
            "update" if n.startswith("k_update") else None
        if key:
            # one launch per kernel: the segmented forward's walk and its reduce add up
            prd, pwr = traffic.get(key, (0.0, 0.0))
            traffic[key] = (prd + rd, pwr + wr)
            try:
                inst[key] = inst.get(key, 0.0) + float(d["smsp__inst_executed.sum"].replace(",", ""))
            except Exception:
                pass
    units = dict(zip(list(csv.reader(io.StringIO(subprocess.run(
        ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))[0],
        list(csv.reader(io.StringIO(subprocess.run(
            ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tj = {}
    for k, (rd, wr) in traffic.items():
        tj[k] = rd * scale.get(units.get("dram__bytes_read.sum", "byte"), 1) + \
            wr * scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
    tj["units"] = "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), capture %s" % tag
    if inst:
        tj["warp_inst"] = inst   # smsp__inst_executed.sum per launch (bench.py: issue fraction)
    with open(os.path.join(ROOT, "profiles", "traffic_%s.json" % cfg), "w") as f:
        json.dump(tj, f, indent=1)
    lines += ["", "DRAM traffic per launch (bytes): " + json.dumps({k: v for k, v in tj.items()
                                                                 if k not in ("units", "warp_inst")})]
    if blog and os.path.exists(blog):
        for line in open(blog):
            if line.startswith("{"):
                lines += ["", "Bench line of the same round:", "", "```", line.strip(), "```"]
    with open(os.path.join(od, "summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
