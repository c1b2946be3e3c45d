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
tl = pk.pcdn_warp_timeline(s.ctx).astype(np.float64).reshape(-1)[: 512 * 8].reshape(512, 8)
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
# warp 0 of each CTA: its chunk partials (A1), wait for the published d_j, records (A2), chunks taken
out["w0_A1_us"] = [round(x, 2) for x in us[-20:, 4]]
out["w0_wait_us"] = [round(x, 2) for x in us[-20:, 5]]
out["w0_scatter_us"] = [round(x, 2) for x in us[-20:, 6]]
out["w0_chunks_per_step"] = [round(x, 3) for x in (tl[:G, 7] / steps)[-20:]]
print(json.dumps(out))
