"""Write tests/golden/fstar.json: the reference optimum F* of each config used by the
Eq.14 stop test (reading Z12).  Calls ONLY oracle/ (and the seeded
generator): no value here comes from the CUDA path.

F* = the oracle's PCDN run far past convergence (the paper uses CDN at eps=1e-8; any
convergent solver reaches the same optimum value).  The KKT residual
(min-norm subgradient) is recorded as evidence of convergence."""
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


def fstar(cfg, loss, max_outer):
    p = synth.config(cfg, loss=loss)
    o = oracle.Oracle(p)
    t = time.time()
    r = o.solve(p.P, seed=p.seed, max_outer=max_outer, trace_cap=0)
    oF = r["outer_F"]
    rel = np.abs(np.diff(oF)) / np.abs(oF[1:])
    sg0, _ = o.min_norm_subgrad(np.zeros(p.n))
    sg, _ = o.min_norm_subgrad(r["w"])
    return dict(F_star=r["F"], outer=int(r["outer"]), last_rel_change=float(rel[-1]) if rel.size else None,
                kkt_l1=float(sg), kkt_l1_at_w0=float(sg0), kkt_ratio=float(sg / max(sg0, 1e-300)),
                null_steps=int(r["null_steps"]), nnz_w=int(np.count_nonzero(r["w"])), P=p.P, seed=p.seed,
                digest=p.digest(), seconds=round(time.time() - t, 1))


if __name__ == "__main__":
    todo = [(1, 0, 400), (1, 1, 400), (2, 1, 1500), (2, 0, 1500)]
    if len(sys.argv) > 1:
        todo = [t for t in todo if str(t[0]) in sys.argv[1:]]
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    res["_citation"] = ("Reference optimum F* for Eq.14 (PAPER.md:398-405, reading Z12), written by "
                        "scripts/make_fstar.py from oracle/ only.")
    for cfg, loss, mo in todo:
        key = f"cfg{cfg}_{'lr' if loss == 0 else 'svm'}"
        res[key] = fstar(cfg, loss, mo)
        print(key, res[key], flush=True)
        json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)
