import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, torch
import paper_1306_4080_b200 as pk
prob = synth.config(2)
arrs = [np.ascontiguousarray(getattr(prob, k), dtype=dt) for k, dt in
        (("col_ptr", np.int64), ("row_idx", np.int32), ("val", np.float32), ("row_ptr", np.int64),
         ("col_idx", np.int32), ("csr_val", np.float32), ("y", np.int8))]
for i in range(4):
    t0 = time.perf_counter()
    st, inf, w = pk.pcdn_train_host(*arrs, prob.c, prob.loss, prob.P, 0.0, 1.0, prob.seed, 1)
    torch.cuda.synchronize()
    print("train_host 1 outer", round(1e3 * (time.perf_counter() - t0), 2), "ms", flush=True)
s = pk.Solver(prob)
for i in range(3):
    t0 = time.perf_counter()
    pk.pcdn_set_launch(s.ctx, 0, 0, 0)
    print("configure", round(1e3 * (time.perf_counter() - t0), 2), "ms", flush=True)
