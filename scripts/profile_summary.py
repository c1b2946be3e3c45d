"""Summarise one GPU pass (scripts/gpu_round.sh) into profiles/<tag>/ for the record:
launch shares from the ncu launch list, key counters of the `ncu --set full` capture of k_step,
the hottest source lines, and the bench JSON line.  Reads gpurun_out/<tag>/ (run here, no GPU).

usage: python scripts/profile_summary.py <tag> [<ncu-rep name> [<launch csv> <summary name> <bench json>]]"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rep_name = sys.argv[2] if len(sys.argv) > 2 else "prof_kstep"
launch_name = sys.argv[3] if len(sys.argv) > 3 else "launches.csv"
summary_name = sys.argv[4] if len(sys.argv) > 4 else "summary.md"
bench_name = sys.argv[5] if len(sys.argv) > 5 else "bench.json"
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles", tag)
os.makedirs(dst, exist_ok=True)
out = []

# 1. launch list -> per-kernel share
lc = os.path.join(src, launch_name)
if os.path.exists(lc):
    hdr, agg = None, defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(lc, errors="replace")):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    out.append("## Launch list (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    out.append("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
    shutil.copy(lc, os.path.join(dst, launch_name))

# 2. full capture counters
rep = os.path.join(src, rep_name + ".ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
            "sass__inst_executed_register_spilling", "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct"]
    out.append("\n## ncu --set full of the top kernel\n")
    for row in rows[2:]:
        kname = row[rows[0].index("Kernel Name")] if "Kernel Name" in rows[0] else "?"
        out.append(f"kernel `{kname[:120]}`\n\n| metric | value | unit |\n|---|---|---|")
        for w in want:
            if w in rows[0]:
                i = rows[0].index(w)
                out.append(f"| {w} | {row[i]} | {rows[1][i]} |")
    srcd = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                          capture_output=True, text=True).stdout
    tmp = os.path.join(dst, "_src.csv")
    open(tmp, "w").write(srcd)
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_source_hot.py"), tmp, "30"],
                         capture_output=True, text=True).stdout
    os.remove(tmp)
    out.append("\n## Hottest source lines (warp-stall samples)\n\n```\n" + hot + "```")

# 3. bench line
bj = os.path.join(src, bench_name)
if os.path.exists(bj):
    lines = [l for l in open(bj) if l.startswith("{")]
    if lines:
        open(os.path.join(dst, bench_name), "w").write(lines[-1])
        b = json.loads(lines[-1])
        out.insert(0, f"# GPU pass {tag}\n\nbench: value {b['value']:.4g} {b['unit']}, ms_per_step {b['ms_per_step']:.3f}, "
                      f"roofline frac {b['roofline']['frac']:.4g} ({b['roofline']['achieved']:.2f} GB/s), "
                      f"clocks {b.get('clocks')}\n")
for extra in ("pytest_gpu.log", "smi.txt"):
    p = os.path.join(src, extra)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, extra))
open(os.path.join(dst, summary_name), "w").write("\n".join(out) + "\n")
print("\n".join(out))
