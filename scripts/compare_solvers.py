"""NEXT #3 (Fig. 3-4, Sec. 5.3): time to the Eq.14 gap on B200 for PCDN
at the configured P, SCDN at the paper's P-bar = 8 (synchronous reading Z27) and CDN
(PCDN with P = 1), all through the C-ABI from w = 0 with the stored F*.

usage: python scripts/compare_solvers.py [--config 2] [--max-outer 400] > profiles/<tag>/compare_cfgN.jsonl"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--max-outer", type=int, default=400)
ap.add_argument("--eps", type=float, default=1e-3)
args = ap.parse_args()
import torch  # noqa: E402

prob = synth.config(args.config)
key = f"cfg{args.config}_{'lr' if prob.loss == 0 else 'svm'}"
fstar = json.load(open(os.path.join(ROOT, "tests", "golden", "fstar.json")))[key]["F_star"]
for name, P, scdn in (("PCDN", prob.P, False), ("SCDN", 8, True), ("CDN", 1, False)):
    s = pk.Solver(prob)
    s.set_launch(3, 0, 100000)
    s.set_scdn(scdn)
    s.solve(P, seed=prob.seed, max_outer=1)   # warm
    s.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = s.solve(P, eps=args.eps, fstar=fstar, seed=prob.seed, max_outer=args.max_outer)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out = dict(config=args.config, solver=name, P=P, status=r["rc"], outer=r["outer_iters"],
               steps=r["steps"], seconds=dt, F=r["F"], gap=(r["F"] - fstar) / fstar,
               us_per_step=1e6 * dt / max(1, r["steps"]))
    print(json.dumps(out), flush=True)
    s.close()
