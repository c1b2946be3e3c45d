"""Stress the single-pass list build (k_prep_lists: ticket + decoupled look-back): many outer
iterations on problems with many tiles, fused vs split list build, repeated -- every run must give
bit-identical w and F traces."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

cases = [("cfg1", synth.config(1), 40), ("cfg3", synth.config(3), 6),
         ("tiny-n513", synth.tiny(5, 64, 513, density=0.2, loss=1, c=2.0, full_cols=3, P=37), 60)]
bad = 0
for name, prob, outer in cases:
    ref = None
    for rep, dbg in enumerate((2, 0, 0, 0)):
        s = pk.Solver(prob)
        pk.pcdn_set_debug(s.ctx, dbg)
        r = s.solve(prob.P, seed=11, max_outer=outer, trace=True)
        cur = (s.w().cpu().numpy().view(np.uint64), r["F_trace"].view(np.uint64), r["q_trace"])
        s.close()
        if ref is None:
            ref = cur
            continue
        same = all(np.array_equal(a, b) for a, b in zip(ref, cur))
        bad += 0 if same else 1
        print(name, "rep", rep, "identical" if same else "DIFFERENT", flush=True)
print("stress done, mismatches:", bad)
