"""Summarise `ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > dump.csv`:
per CUDA source line, warp-stall samples (with the top stall reasons) and executed warp
instructions (top N).  `--sass` lists the hottest SASS instructions instead."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
sass = "--sass" in sys.argv
hdr, lines, fn = None, [], None
for r in csv.reader(open(path, errors="replace")):
    if not r:
        continue
    if r[0] == "Function Name":
        fn = r[1]
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    is_src = r[0].isdigit() and r[2] == "-"
    if sass == is_src:
        continue
    def num(i):
        try:
            return float(r[i] or 0)
        except (ValueError, IndexError):
            return 0.0
    reasons = {hdr[i][6:]: num(i) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}
    label = (r[0] + " " + r[1].strip())[:100] if not sass else (r[2] + " " + r[3].strip())[:100]
    lines.append((label, num(4), num(7), reasons))
tot = sum(l[1] for l in lines) or 1
toti = sum(l[2] for l in lines) or 1
print(f"{fn}\ntotal stall samples {tot:.0f}, warp instructions {toti:.4g}")
for label, s, ins, rs in sorted(lines, key=lambda l: -l[1])[:top]:
    big = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
    why = " ".join(f"{k}={100 * v / max(s, 1):.0f}%" for k, v in big if v > 0)
    print(f"{100 * s / tot:5.1f}% smp {100 * ins / toti:5.1f}% ins | {label:100s} | {why}")
