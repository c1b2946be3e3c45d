"""Small cases of every launch mode for the checked build (libpcdn_checked.so, device-side bounds and
protocol checks; compute-sanitizer is closed on this pool): one bundle step from an injected state
and a two-outer-iteration solve per mode and loss on a tiny fixture and on config 1, plus SCDN,
elastic net, Lasso, the dense kernel, the sample-sharded step and the one-call host API.  Prints one
line per case; exits non-zero if a result leaves the oracle's north-star bars (a failed check traps
the kernel and the CUDA error ends the run).

usage: PCDN_LIB=paper_1306_4080_b200/libpcdn_checked.so python scripts/checked_cases.py [--quick]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

quick = "--quick" in sys.argv
bad = 0


def check(name, gs, os_, w):
    global bad
    ok = abs(gs["F"] - os_["F"]) <= 1e-6 * abs(os_["F"]) and np.max(np.abs(w - os_["w"])) <= 1e-5
    bad += 0 if ok else 1
    print(f"{name}: F {gs['F']:.12g} oracle {os_['F']:.12g} {'ok' if ok else 'MISMATCH'}", flush=True)


def run(name, prob, launch, P, outer=2, setup=None, oracle_kw=None):
    s = pk.Solver(prob)
    if launch:
        s.set_launch(*launch)
    if setup:
        setup(s)
    o = oracle.Oracle(prob, **(oracle_kw or {}))
    w = np.random.default_rng(1).normal(size=prob.n) * 0.2 * (np.random.default_rng(2).random(prob.n) < 0.3)
    B = np.random.default_rng(3).choice(prob.n, size=min(P, prob.n), replace=False).astype(np.int32)
    s.set_w(w)
    r = s.step(B)
    ro = o.step(w, B)
    print(f"{name}: step q {r['q']} oracle {ro['q']}", flush=True)
    s.reset()
    gs = s.solve(P, seed=3, max_outer=outer)
    check(name, gs, o.solve(P, seed=3, max_outer=outer), s.w().cpu().numpy())
    s.close()


tiny = [synth.tiny(5, 150, 30, density=0.1, loss=l, c=3.0, full_cols=2, dense_rows=1, P=7) for l in (0, 1)]
cfgs = tiny if quick else tiny + [synth.config(1, loss=l) for l in (0, 1)]
for prob in cfgs:
    for launch in ((1, 4, 0), (1, 16, 2), (2, 3, 1), (2, 0, 0), (3, 0, 0), (3, 4, 1, 2), (5, 3, 2)):
        if len(launch) == 4:
            def setup(s, cap=launch[3]):
                pk.pcdn_set_resident_cap(s.ctx, cap)
            run(f"{prob.name} mode {launch}", prob, launch[:3], prob.P, setup=setup)
        else:
            run(f"{prob.name} mode {launch}", prob, launch, prob.P)
dense = synth.tiny(31, 40, 60, density=1.0, loss=0, c=4.0, P=20)
run("dense mode 4", dense, (4, 3, 0), 20)
run("scdn", tiny[0], (3, 0, 100000), 8, setup=lambda s: s.set_scdn(True))
run("elastic", tiny[1], (2, 3, 1), 7, setup=lambda s: s.set_elastic(1.5), oracle_kw={"mu": 1.5})
lasso = synth.regression(synth.tiny(5, 150, 30, density=0.1, c=0.7, P=7), noise=0.2, support=5)
run("lasso", lasso, (2, 3, 1), 7)
ss = pk.ShardedSolver(tiny[0])
r = ss.solve(7, seed=4, max_outer=2, trace=True)
check("sharded world 1", r, oracle.Oracle(tiny[0]).solve(7, seed=4, max_outer=2), ss.w().cpu().numpy())
ss.close()
a = [np.ascontiguousarray(getattr(tiny[1], k), dtype=dt) for k, dt in
     (("col_ptr", np.int64), ("row_idx", np.int32), ("val", np.float32), ("y", np.int8))]
st, inf, w = pk.pcdn_train_host(a[0], a[1], a[2], None, None, None, a[3], tiny[1].c, tiny[1].loss, 7, 0.0, 1.0, 3, 2)
check("train_host", {"F": inf.F}, oracle.Oracle(tiny[1]).solve(7, seed=3, max_outer=2), w)
print("cases with mismatches:", bad, flush=True)
sys.exit(1 if bad else 0)
