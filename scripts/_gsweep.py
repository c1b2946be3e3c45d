import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1306_4080_b200 as pk
for cfg in (1, 2, 3):
    prob = synth.config(cfg)
    s = pk.Solver(prob)
    for G in (4, 8, 16):
        try:
            s.set_launch(3, G, 0)
            s.reset(); s.solve(prob.P, seed=prob.seed, max_outer=1)
            ts = []
            for rep in range(3):
                s.reset(); torch.cuda.synchronize(); t0 = time.perf_counter()
                r = s.solve(prob.P, seed=prob.seed, max_outer=2)
                torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
            print(f"cfg{cfg} G={G}: {1e6 * min(ts) / r['steps']:.2f} us/step (2 outer, wall)", flush=True)
        except Exception as e:
            print(f"cfg{cfg} G={G}: {e}")
    s.close()
