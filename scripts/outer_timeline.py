"""GPU timeline of one solve (torch.profiler / CUPTI activity records): every kernel and copy of
the library with its start and duration, and the idle gaps between them, to see what an outer
iteration costs beyond its step launch.

usage: python scripts/outer_timeline.py <cfg> [--outer K] [--out file.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("--outer", type=int, default=3)
ap.add_argument("--eps", type=float, default=0.0)
ap.add_argument("--out", default="")
args = ap.parse_args()
prob = synth.config(args.cfg)
s = pk.Solver(prob)
for _ in range(2):
    s.reset()
    s.solve(prob.P, seed=prob.seed, max_outer=args.outer, eps=0.0)
s.reset()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pk.pcdn_reset(s.ctx)   # as bench.py's timed solve: from w = 0
    st_, inf_ = pk.pcdn_solve(s.ctx, prob.P, 0.0, prob.seed, args.outer)
    torch.cuda.synchronize()
r = inf_.as_dict()
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA or "cuda" in str(e.device_type).lower():
        ev.append((e.time_range.start, e.time_range.end, e.name))
ev.sort()
t0 = ev[0][0] if ev else 0
rows = []
prev_end = None
for st, en, name in ev:
    gap = None if prev_end is None else st - prev_end
    rows.append({"t_us": round(st - t0, 1), "dur_us": round(en - st, 1), "gap_us": None if gap is None else round(gap, 1),
                 "name": name[:70]})
    prev_end = en if prev_end is None else max(prev_end, en)
for x in rows:
    print(f"{x['t_us']:10.1f} {x['dur_us']:9.1f} {'' if x['gap_us'] is None else x['gap_us']:>8} {x['name']}")
tot = (ev[-1][1] - t0) if ev else 0
busy = sum(en - st for st, en, _ in ev)
print(json.dumps({"cfg": args.cfg, "outer": r["outer_iters"], "span_us": round(tot, 1), "sum_dur_us": round(busy, 1),
                  "t_gpu_ms": r["t_gpu_ms"], "t_step_kernel_ms": r["t_step_kernel_ms"]}))
if args.out:
    json.dump(rows, open(args.out, "w"), indent=0)
