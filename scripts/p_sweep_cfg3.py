"""Config 3 (news20-shaped, BASELINE.json configs[2]) at P in {1, 64, 1024, 8192}: time to the Eq.14
gap 1e-3 on the GPU (auto launch mode), steps, outer iterations, step time -- the prescribed sweep
(Fig. 2 / Table 3 analog).  One JSON line per P."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "fstar.json")))
fstar = g["cfg3_lr"]["F_star"]
prob = synth.config(3)
s = pk.Solver(prob)
Ps = [a for a in sys.argv[1:] if not a.startswith("--")]
for P in [int(x) for x in (Ps[0] if Ps else "1,64,1024,8192").split(",")]:
    s.reset()
    s.solve(P, eps=1e-3, seed=prob.seed, max_outer=200, fstar=fstar)   # warm
    s.reset()
    r = s.solve(P, eps=1e-3, seed=prob.seed, max_outer=200, fstar=fstar)
    print(json.dumps({"cfg": 3, "P": P, "rc": r["rc"], "outer": r["outer_iters"], "steps": r["steps"],
                      "time_to_gap_ms": r["t_gpu_ms"], "step_us": 1e3 * r["t_step_kernel_ms"] / r["steps"],
                      "mode": pk.pcdn_phase_cycles(s.ctx)[1], "F": r["F"], "gap": r["gap"]}), flush=True)
s.close()
if "--oracle-p1" in sys.argv:   # the CPU oracle's full solve at P = 1 (CDN order), one pinned core
    import time
    import oracle
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass
    t = time.perf_counter()
    r = oracle.Oracle(prob).solve(1, eps=1e-3, fstar=fstar, seed=prob.seed, max_outer=200, trace_cap=0)
    print(json.dumps({"cfg": 3, "P": 1, "impl": "oracle (CPU, 1 core)", "rc": r["rc"], "outer": r["outer"],
                      "steps": r["steps"], "time_to_gap_ms": 1e3 * (time.perf_counter() - t),
                      "F": r["F"], "gap": r["gap"]}), flush=True)
