"""Cost of the sample-sharded step (NEXT #2) on one B200 with one rank: host-driven phases
(4 C-ABI calls, 2 cross-rank sums, a host decision per step) against the fused persistent
kernels, one outer iteration of the given config.  With more GPUs the per-rank shard shrinks;
the per-step latency floor (launches + collectives + host decision) stays."""
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
ap.add_argument("--outer", type=int, default=1)
args = ap.parse_args()
import torch  # noqa: E402

prob = synth.config(args.config)
s = pk.Solver(prob)
s.solve(prob.P, seed=prob.seed, max_outer=1)
s.reset()
torch.cuda.synchronize()
t0 = time.perf_counter()
r = s.solve(prob.P, seed=prob.seed, max_outer=args.outer)
torch.cuda.synchronize()
t_fused = time.perf_counter() - t0
s.close()
ss = pk.ShardedSolver(prob)
torch.cuda.synchronize()
t0 = time.perf_counter()
rs = ss.solve(prob.P, seed=prob.seed, max_outer=args.outer)
torch.cuda.synchronize()
t_sh = time.perf_counter() - t0
print(json.dumps(dict(config=args.config, P=prob.P, outer=args.outer, steps=rs["steps"],
                      fused_ms=1e3 * t_fused, sharded_world1_ms=1e3 * t_sh,
                      fused_us_per_step=1e6 * t_fused / r["steps"], sharded_us_per_step=1e6 * t_sh / rs["steps"],
                      F_fused=r["F"], F_sharded=rs["F"])))
