"""DRAM traffic per launch of the step kernel from an ncu capture, into profiles/traffic.json.

bench.py reports roofline.traffic from this file for the exact (config, loss, P, kernel) it times.
The capture is `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:<kernel> --csv ... python bench.py --config C --steps 1 --warmup 0 ...` (every launch of
one solve); the entry is the mean over the captured launches.

usage: python scripts/traffic_from_ncu.py <ncu csv> <key> <source note>"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, key, note = sys.argv[1], sys.argv[2], sys.argv[3]
per = defaultdict(dict)
units = {}
hdr = None
for r in csv.reader(open(path, errors="replace")):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d.get("Metric Name")
    if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "msecond": 1e-3, "second": 1.0}[d["Metric Unit"]]
        per[d["ID"]][name] = float(d["Metric Value"].replace(",", "")) * scale
# (a launch queued after the outer iteration that ended the solve exits at once: not a step launch)
launches = [v for v in per.values() if len(v) == 3 and v["gpu__time_duration.sum"] > 1e-3]
if not launches:
    raise SystemExit("no complete launches in " + path)
rd = sum(v["dram__bytes_read.sum"] for v in launches) / len(launches)
wr = sum(v["dram__bytes_write.sum"] for v in launches) / len(launches)
t = sum(v["gpu__time_duration.sum"] for v in launches) / len(launches)
out_path = os.path.join(ROOT, "profiles", "traffic.json")
try:
    allv = json.load(open(out_path))
except (OSError, ValueError):
    allv = {}
allv[key] = {"dram_bytes_per_launch": rd + wr, "dram_read_per_launch": rd, "dram_write_per_launch": wr,
             "launches": len(launches), "mean_launch_s_under_ncu": t, "source": note}
json.dump(allv, open(out_path, "w"), indent=1, sort_keys=True)
print(key, json.dumps(allv[key]))
