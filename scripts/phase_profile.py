"""Per-phase time of the persistent step kernel (profiling mode, CTA 0 clock64 counters)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

NAMES = ["A rest", "sync1", "C1 touched set", "C2 fold+LS loops", "C3 reduce+xbar", "decide",
         "commit", "sync3", "A light", "A' search", "A' rounds", "A' gridsync"]
# k_step_sparse (launch modes 1, 2): its SP_MARK slots
SPARSE_NAMES = ["A2 heavy scatter", "sync1", "C1 touched set", "fold+LS", "sync2", "decide", "commit", "sync3",
                "A light+medium", "A1 heavy chunks"]

# k_step_dense (launch mode 4): its DPROF slots (in order along a step)
DENSE_NAMES = ["B1 fence+prefetch issue", "B1 wait", "D finish cols", "B2", "X d'x", "LS", "G", "-", "tile wait",
               "resolve tail(commit+F)", "B1 arrive", "X dk load+or", "X chunks", "resolve decide", "resolve commit z/w"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--P", type=int, default=None)
ap.add_argument("--modes", default="1,2")
ap.add_argument("--ctas", default="0")
ap.add_argument("--outer", type=int, default=2)
ap.add_argument("--mhz", type=float, default=1965.0)
args = ap.parse_args()
prob = synth.config(args.config)
P = args.P or prob.P
s = pk.Solver(prob)
res = {}
for mode in [int(m) for m in args.modes.split(",")]:
    for ctas in [int(c) for c in args.ctas.split(",")]:
        if mode == 1 and ctas > 16:
            continue
        s.set_launch(mode, ctas, 0)
        s.reset()
        s.solve(P, seed=prob.seed, max_outer=1)          # warm
        s.reset()
        pk.pcdn_set_profile(s.ctx, 1)
        r = s.solve(P, seed=prob.seed, max_outer=args.outer)
        cyc, m = pk.pcdn_phase_cycles(s.ctx)
        pk.pcdn_set_profile(s.ctx, 0)
        steps = r["steps"]
        names = SPARSE_NAMES if m in (1, 2) else DENSE_NAMES if m == 4 else NAMES
        us = cyc[:len(names)] / steps / args.mhz
        key = f"mode{m}_ctas{ctas}"
        res[key] = dict(step_us_kernel=r["t_step_kernel_ms"] * 1e3 / steps, phases_us=dict(zip(names, us.round(3).tolist())),
                        steps=steps)
        print(key, f"kernel {r['t_step_kernel_ms']*1e3/steps:.2f} us/step |",
              " ".join(f"{n}={u:.2f}" for n, u in zip(names, us)), flush=True)
print(json.dumps(res))
