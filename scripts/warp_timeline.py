"""Per-warp timeline of the cluster-resident step kernel (profiling mode 2, CTA 0): for each of 14
points of a step, min / median / max over the 16 warps of the cycles since the step began
(earliest warp at point 0), averaged over steps 2..15 of one outer iteration."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

PTS = ["0 step start", "1 light cols done", "2 heavy done", "3 counts sent", "4 M0 done", "5 lazy commit",
       "6 M1 done", "7 linked", "8 fold+LS loops", "9 CTA reduce", "10 sent+staged", "11 M2 done",
       "12 decided", "13 commit tail", "14 link+full cols", "15 compaction"]
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--P", type=int, default=None)
args = ap.parse_args()
prob = synth.config(args.config)
s = pk.Solver(prob)
s.set_launch(3, 0, 0)
P = args.P or prob.P
s.solve(P, seed=prob.seed, max_outer=1)
s.reset()
pk.pcdn_set_profile(s.ctx, 2)
s.solve(P, seed=prob.seed, max_outer=1)
tl = pk.pcdn_warp_timeline(s.ctx).astype(np.float64)   # [step][warp][pt]
pk.pcdn_set_profile(s.ctx, 0)
rel = []
for st in range(2, 16):
    t0 = tl[st, :, 0][tl[st, :, 0] > 0].min()
    rel.append(np.where(tl[st] > 0, tl[st] - t0, np.nan))
rel = np.array(rel)   # [steps][warp][pt]
nxt = []
for st in range(2, 15):
    nxt.append(tl[st + 1, :, 0][tl[st + 1, :, 0] > 0].min() - tl[st, :, 0][tl[st, :, 0] > 0].min())
print(f"cfg{args.config} P={P}: step period {np.mean(nxt):.0f} cycles ({np.mean(nxt) / 1965:.2f} us at 1965 MHz)")
print(f"{'point':22s} {'min':>8s} {'median':>8s} {'max':>8s} {'warp0':>8s} {'warp15':>8s}   (cycles since step start, mean over steps)")
for p, name in enumerate(PTS):
    v = rel[:, :, p]
    print(f"{name:22s} {np.nanmean(np.nanmin(v, 1)):8.0f} {np.nanmean(np.nanmedian(v, 1)):8.0f} {np.nanmean(np.nanmax(v, 1)):8.0f}"
          f" {np.nanmean(v[:, 0]):8.0f} {np.nanmean(v[:, -1]):8.0f}")
d78 = np.nanmedian(rel[:, :, 8] - rel[:, :, 7], 0)
d01 = np.nanmedian(rel[:, :, 1] - rel[:, :, 0], 0)
print("per-warp median cycles, fold+LS pass (7->8):", " ".join(f"{v:.0f}" for v in d78))
print("per-warp median cycles, light columns (0->1):", " ".join(f"{v:.0f}" for v in d01))
