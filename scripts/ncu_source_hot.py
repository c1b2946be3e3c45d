"""Summarise `ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > dump.csv`:
per CUDA source line, warp-stall samples and executed warp instructions (top N)."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr, lines, fn = None, [], None
for r in csv.reader(open(path, errors="replace")):
    if not r:
        continue
    if r[0] == "Function Name":
        fn = r[1]
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < 8 or r[2] != "-":
        continue
    def num(i):
        try:
            return float(r[i] or 0)
        except ValueError:
            return 0.0
    lines.append((int(r[0]), r[1].strip()[:100], num(4), num(7)))
tot = sum(l[2] for l in lines) or 1
toti = sum(l[3] for l in lines) or 1
print(f"{fn}\ntotal stall samples {tot:.0f}, warp instructions {toti:.4g}")
for ln, src, s, ins in sorted(lines, key=lambda l: -l[2])[:top]:
    print(f"{ln:5d} {100*s/tot:5.1f}% smp {100*ins/toti:5.1f}% ins | {src}")
