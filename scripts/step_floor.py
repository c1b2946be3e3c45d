"""Per-step floor of each step kernel (SURVEY.md 8(d) "the measured per-step floor: the time of an
all-empty bundle step"): a problem whose columns are all empty but one (s = 20,000 samples,
n = 200,000 features), solved with P = 1 for one outer iteration -- 200,000 bundle steps, all but one
with an empty bundle (d_j = 0, T empty, q = 0) -- in each launch mode; the step kernel's CUDA-event
time / steps is the floor of its per-step exchange chain.  One JSON line per mode.

usage: python scripts/step_floor.py [--P 1] [--modes 1,2,3,5]"""
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
ap.add_argument("--P", type=int, default=1)
ap.add_argument("--modes", default="1,2,3,5")
ap.add_argument("--s", type=int, default=20000)
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--profile", action="store_true", help="phase cycles of CTA 0 (needs PCDN_LIB=.../libpcdn_prof.so)")
args = ap.parse_args()
s_, n_ = args.s, args.n
rng = np.random.default_rng(0)
rows = np.sort(rng.choice(s_, size=50, replace=False)).astype(np.int32)
col_ptr = np.zeros(n_ + 1, dtype=np.int64)
col_ptr[1:] = rows.size   # column 0 holds the 50 nonzeros, every other column is empty
val = np.full(rows.size, 0.5, dtype=np.float32)
y = np.where(rng.random(s_) < 0.5, 1, -1).astype(np.int8)
prob = synth.Problem(name="floor", s=s_, n=n_, col_ptr=col_ptr, row_idx=rows, val=val,
                     row_ptr=np.zeros(s_ + 1, dtype=np.int64), col_idx=np.zeros(0, dtype=np.int32),
                     csr_val=np.zeros(0, dtype=np.float32), y=y, c=1.0, loss=0, P=args.P, seed=0)
rp = np.zeros(s_ + 1, dtype=np.int64)
np.add.at(rp, rows + 1, 1)
prob.row_ptr = np.cumsum(rp).astype(np.int64)
prob.col_idx = np.zeros(rows.size, dtype=np.int32)
prob.csr_val = val.copy()
s = pk.Solver(prob)
for mode in [int(m) for m in args.modes.split(",")]:
    try:
        s.set_launch(mode, 0, 0)
    except pk.PCDNError as e:
        print(json.dumps({"mode": mode, "error": str(e)}), flush=True)
        continue
    s.reset()
    s.solve(args.P, seed=1, max_outer=1)
    s.reset()
    if args.profile:
        pk.pcdn_set_profile(s.ctx, 1)
    r = s.solve(args.P, seed=1, max_outer=1)
    cyc, used = pk.pcdn_phase_cycles(s.ctx)
    if args.profile:
        pk.pcdn_set_profile(s.ctx, 0)
    out = {"mode_req": mode, "mode_used": used, "P": args.P, "steps": r["steps"],
           "step_us": 1e3 * r["t_step_kernel_ms"] / r["steps"], "nnz": int(r["nnz_processed"])}
    if args.profile:
        out["phase_cycles"] = (cyc / r["steps"]).round().tolist()
    print(json.dumps(out), flush=True)
s.close()
