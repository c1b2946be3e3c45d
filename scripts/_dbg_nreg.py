import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, oracle
import paper_1306_4080_b200 as pk
TINY1 = dict(seed=2, s=70, n=33, density=0.2, empty_cols=4, dup_cols=2)
for launch in [(1, 4, 1), (2, 3, 2), (1, 1, 0), (2, 0, 1)]:
    prob = synth.tiny(loss=0, c=3.0, P=5, **TINY1)
    rng = np.random.default_rng(101)
    s = pk.Solver(prob); s.set_launch(*launch)
    o = oracle.Oracle(prob)
    bad = 0
    for rep in range(3):
        w = rng.normal(size=prob.n) * 0.5 * rep * (rng.random(prob.n) < 0.3)
        for P in [1, 2, 5, 16]:
            B = rng.choice(prob.n, size=min(P, prob.n), replace=False).astype(np.int32)
            s.set_w(w)
            g = s.step(B)
            r = o.step(w, B)
            T = r["T"]
            gT = g["T"]
            if not np.array_equal(np.sort(gT), T):
                print("T mismatch", launch, P); bad += 1; continue
            gd = dict(zip(g["T"].tolist(), g["dx"].tolist()))
            od = dict(zip(T.tolist(), r["dx"].tolist()))
            X = prob.dense()
            for i in T.tolist():
                if abs(gd[i] - od[i]) > 1e-9 * (1 + abs(od[i])):
                    nrec = int(np.sum(X[i, B] != 0))
                    print("launch", launch, "P", P, "sample", i, "gpu", gd[i], "ora", od[i], "records", nrec)
                    bad += 1
    print("launch", launch, "bad", bad)
