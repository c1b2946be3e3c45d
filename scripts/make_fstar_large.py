"""F* for the large configs (3, 4, 5) by the CPU oracle, for the Eq.14 stop test (PAPER.md:398-405,
reading Z12).  Calls ONLY oracle/ (and the seeded generator): no value comes from the CUDA path.

The oracle's PCDN is run in chunks of `chunk` outer iterations, each warm-started from the
previous w with a fresh partition stream (seed + chunk index; any convergent schedule reaches the
same optimum value), until the objective changes by less than `tol` (relative)
over a whole chunk or the time budget runs out.  The KKT residual (min-norm subgradient,
SPEC.md:145-153) is recorded as evidence of convergence.

usage: python scripts/make_fstar_large.py <cfg> <loss 0|1> [tol] [budget_s] [chunk]"""
import fcntl
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fstar.json")


def main():
    cfg, loss = int(sys.argv[1]), int(sys.argv[2])
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-10
    budget = float(sys.argv[4]) if len(sys.argv) > 4 else 6 * 3600
    chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 10
    key = f"cfg{cfg}_{'lr' if loss == 0 else 'svm'}"
    p = synth.config(cfg, loss=loss)
    o = oracle.Oracle(p)
    t0 = time.time()
    w = np.zeros(p.n)
    F_prev, outer, hist = None, 0, []
    while True:
        r = o.solve(p.P, seed=p.seed + 1000003 * (outer // chunk), max_outer=chunk, w0=w, trace_cap=0)
        w = r["w"]
        outer += r["outer"]
        F = r["F"]
        rel = abs(F_prev - F) / abs(F) if F_prev is not None else float("inf")
        hist.append((outer, F, rel, round(time.time() - t0, 1)))
        print(key, outer, repr(F), rel, round(time.time() - t0, 1), flush=True)
        F_prev = F
        if rel < tol or time.time() - t0 > budget:
            break
    sg0, _ = o.min_norm_subgrad(np.zeros(p.n))
    sg, _ = o.min_norm_subgrad(w)
    res = dict(F_star=F, outer=outer, last_rel_change=rel, kkt_l1=float(sg), kkt_l1_at_w0=float(sg0),
               kkt_ratio=float(sg / max(sg0, 1e-300)), nnz_w=int(np.count_nonzero(w)), P=p.P, seed=p.seed,
               digest=p.digest(), seconds=round(time.time() - t0, 1), chunk=chunk, tol=tol,
               converged=bool(rel < tol), method="oracle PCDN, warm-started chunks (scripts/make_fstar_large.py)")
    with open(OUT + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        cur = json.load(open(OUT)) if os.path.exists(OUT) else {}
        cur[key] = res
        json.dump(cur, open(OUT, "w"), indent=1, sort_keys=True)
    print("wrote", key, res, flush=True)


if __name__ == "__main__":
    main()
