"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump: per CUDA source line,
warp-stall samples and executed instructions (top N)."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = None
lines = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r:
        continue
    if r[0] and r[0].isdigit():
        d = dict(zip(hdr[4:], r[4:]))
        def num(k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0
        lines.append((int(r[0]), r[1].strip()[:90], num("Warp Stall Sampling (All Samples)"),
                      num("Instructions Executed"), {k: num(k) for k in hdr[4:] if k.startswith("stall_") and "Not Issued" not in k}))
tot = sum(l[2] for l in lines) or 1
toti = sum(l[3] for l in lines) or 1
print(f"total samples {tot:.0f}, instructions {toti:.3g}")
for ln, src, s, ins, st in sorted(lines, key=lambda l: -l[2])[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{ln:5d} {100*s/tot:5.1f}% smp {100*ins/toti:5.1f}% ins | {src:90s} | " + " ".join(f"{k[6:]}={v:.0f}" for k, v in big))
