"""P sweep on B200 (Fig. 1 and Fig. 2 analogs): for each
bundle size P, solve the workload from w0 = 0 to the Eq.14 gap eps with the CUDA path and record
the outer iterations, the bundle steps T_eps (inner iterations, Theorem 2's T), the mean accepted
line-search index q, device time, and E[lambda_bar(B)]/P (Lemma 1(a)), which Eq.15 says
T_eps^up is proportional to (times n).  Prints one JSON line per P.

usage: python scripts/p_sweep.py --config 2 --P 16,64,256,1024,4096 [--eps 1e-3]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402
from paper_1306_4080_b200 import diagnostics as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--loss", type=int, default=None)
ap.add_argument("--P", default="16,64,256,1024,4096")
ap.add_argument("--eps", type=float, default=1e-3)
ap.add_argument("--max-outer", type=int, default=2000)
args = ap.parse_args()
prob = synth.config(args.config, loss=args.loss)
g = json.load(open(os.path.join(ROOT, "tests", "golden", "fstar.json")))
fstar = g[f"cfg{args.config}_{'lr' if prob.loss == 0 else 'svm'}"]["F_star"]
lam = dg.column_sq_norms(prob.col_ptr, prob.val)
s = pk.Solver(prob)
for P in [int(x) for x in args.P.split(",")]:
    b = -(-prob.n // P)
    s.reset()
    s.solve(P, eps=0.0, seed=prob.seed, max_outer=1)   # warm-up
    s.reset()
    trace = args.max_outer * b <= 4_000_000
    r = s.solve(P, eps=args.eps, seed=prob.seed, max_outer=args.max_outer, fstar=fstar, trace=trace)
    out = {"config": args.config, "loss": prob.loss, "P": P, "rc": r["rc"], "outer": r["outer_iters"],
           "T_eps_steps": r["steps"], "gap": r["gap"], "kernel_ms": r["t_step_kernel_ms"], "gpu_ms": r["t_gpu_ms"],
           "step_us": 1e3 * r["t_step_kernel_ms"] / max(1, r["steps"]),
           "E_lambda_bar": dg.expected_lambda_max(lam, P), "E_lambda_bar_over_P": dg.expected_lambda_max(lam, P) / P}
    if trace:
        q = r["q_trace"]
        out["mean_q"] = float(np.mean(q[q >= 0])) if q.size else None
        out["null_steps"] = int(np.sum(q < 0))
    print(json.dumps(out), flush=True)
