"""GPU timeline (CUPTI via torch.profiler) of one pcdn_train_host call on config 2: copies, kernels
and gaps, to see what the end-to-end path adds to the device solve."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = synth.config(cfg)
g = json.load(open(os.path.join(ROOT, "tests", "golden", "fstar.json")))
fstar = g[f"cfg{cfg}_{'lr' if prob.loss == 0 else 'svm'}"]["F_star"]
pin = {}
for name, dt in (("col_ptr", np.int64), ("row_idx", np.int32), ("val", np.float32), ("row_ptr", np.int64),
                 ("col_idx", np.int32), ("csr_val", np.float32), ("y", np.int8)):
    a = np.ascontiguousarray(getattr(prob, name), dtype=dt)
    t = torch.empty(a.shape, dtype=getattr(torch, np.dtype(dt).name), pin_memory=True)
    t.numpy()[...] = a
    pin[name] = t
w_host = torch.empty(prob.n, dtype=torch.float64, pin_memory=True)
stream = torch.cuda.Stream()


def once():
    return pk.pcdn_train_host(*(pin[k].numpy() for k in ("col_ptr", "row_idx", "val", "row_ptr", "col_idx", "csr_val",
                                                         "y")), prob.c, prob.loss, prob.P, 1e-3, fstar, prob.seed, 1000,
                              stream=stream, w_out=w_host.numpy())


for _ in range(3):
    once()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    once()
    torch.cuda.synchronize()
rt = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type != torch.autograd.DeviceType.CUDA and e.name.startswith("cuda"))
if rt:
    r0 = rt[0][0]
    tot = {}
    for st, en, name in rt:
        tot[name] = tot.get(name, [0, 0.0])
        tot[name][0] += 1
        tot[name][1] += en - st
    print("runtime API calls (count, total us):")
    for k, v in sorted(tot.items(), key=lambda x: -x[1][1])[:20]:
        print(f"  {v[1]:10.1f} {v[0]:6d} {k}")
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA)
t0 = ev[0][0]
prev = None
agg = {}
for st, en, name in ev:
    gap = "" if prev is None else f"{st - prev:8.1f}"
    print(f"{st - t0:10.1f} {en - st:9.1f} {gap:>8} {name[:60]}")
    prev = en if prev is None else max(prev, en)
    k = name.split("(")[0][:40]
    agg[k] = agg.get(k, 0.0) + (en - st)
print("span_us", round(ev[-1][1] - t0, 1))
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
    print(f"{v:10.1f} {k}")
