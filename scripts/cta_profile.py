"""Per-CTA phase times of the sparse HBM-state step kernel (profiling mode 2): for each CTA of the
launch, the mean cycles per step of phase A (g/h/d + records, until all its warps are done), the
touched-set build, touched-set build + fold + line-search partials, and the mean touched samples --
to locate the CTAs that hold the grid barriers.

usage: python scripts/cta_profile.py <cfg> [--loss L] [--P P] [--mode 2]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("--loss", type=int, default=None)
ap.add_argument("--P", type=int, default=None)
ap.add_argument("--mode", type=int, default=2)
ap.add_argument("--mhz", type=float, default=1965.0)
args = ap.parse_args()
prob = synth.config(args.cfg, loss=args.loss)
s = pk.Solver(prob)
s.set_launch(args.mode, 0, 0)
P = args.P or prob.P
s.solve(P, seed=prob.seed, max_outer=1)
s.reset()
pk.pcdn_set_profile(s.ctx, 2)
r = s.solve(P, seed=prob.seed, max_outer=1)
steps = r["steps"]
tl = pk.pcdn_warp_timeline(s.ctx).astype(np.float64).reshape(-1)[: 256 * 16].reshape(256, 16)
pk.pcdn_set_profile(s.ctx, 0)   # (zeroes the counters)
G = int(np.count_nonzero(tl[:, 0]))
us = tl[:G] / steps / args.mhz
out = {"cfg": args.cfg, "P": P, "mode": args.mode, "G": G, "steps": steps, "step_us": r["t_step_kernel_ms"] * 1e3 / steps}
for k, name in ((0, "A_us"), (3, "C1_us"), (1, "C1+fold+LS_us")):
    v = us[:, k]
    out[name] = {"min": round(v.min(), 3), "median": round(float(np.median(v)), 3), "max": round(v.max(), 3),
                 "argmax": int(v.argmax())}
out["touched_per_cta"] = {"median": float(np.median(tl[:G, 2] / steps)), "max": float((tl[:G, 2] / steps).max())}
out["A_us_by_cta"] = [round(x, 2) for x in us[:, 0]]
# per-CTA points of phase A (cycles since the step began, mean per step): lane sweep done, medium
# columns done, heavy chunks reduced; medium columns per step
for k, name in ((9, "lane_done_us_by_cta"), (10, "medium_done_us_by_cta"), (11, "A1_done_us_by_cta")):
    out[name] = [round(x, 2) for x in us[:, k]]
out["medium_cols_by_cta"] = [round(x, 2) for x in tl[:G, 12] / steps]
# thread 0 of each light CTA, its lane columns: cycles until the column descriptor, the rows, the
# gathered factors are in registers, and the emits issued (per lane column it handled)
lc = tl[:G, 8]
sel = lc > 0
for k, name in ((4, "colinfo"), (5, "rows"), (6, "coef"), (7, "finish+emit")):
    out["lane_col_cycles_" + name] = round(float(np.sum(tl[:G, k][sel]) / np.sum(lc[sel])), 1)
out["lane_cols_per_step_thread0"] = round(float(np.mean(lc[sel]) / steps), 3)
print(json.dumps(out))
