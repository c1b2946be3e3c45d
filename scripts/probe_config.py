"""Per-step time and kernel bandwidth of the step kernel for one config at several bundle sizes P
and launch modes (fixed outer iterations, no stop test).  One process: the data is generated
once.  Prints one JSON line per (P, mode).

usage: python scripts/probe_config.py <cfg> [loss] --P 4096,100000 --modes 0,1,2 --outer 1"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import synth  # noqa: E402
import paper_1306_4080_b200 as pk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("--loss", type=int, default=None)
ap.add_argument("--P", default="")
ap.add_argument("--modes", default="0")
ap.add_argument("--outer", type=int, default=1)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--heavy", type=int, default=0, help="heavy_len launch knob (0 = keep)")
ap.add_argument("--ctas", default="0", help="comma list of CTA counts (launch knob; 0 = all co-resident)")
ap.add_argument("--debug", default="0", help="comma list of pcdn_set_debug values (e.g. 8: no next-step staging)")
ap.add_argument("--l2", type=int, default=0, help="persisting-L2 window of the HBM-state kernels (pcdn_set_l2_persist; the library default is off)")
args = ap.parse_args()
t0 = time.time()
prob = synth.config(args.cfg, loss=args.loss)
print(json.dumps({"generated_s": round(time.time() - t0, 1), "s": prob.s, "n": prob.n, "nnz": prob.nnz}), flush=True)
s = pk.Solver(prob)
pk.pcdn_set_l2_persist(s.ctx, args.l2)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
Ps = [int(x) for x in args.P.split(",") if x] or [prob.P]
for P, mode, ctas, dbg in [(P, int(m), int(g), int(d)) for P in Ps for m in args.modes.split(",") for g in args.ctas.split(",")
                           for d in args.debug.split(",")]:
    if True:
        pk.pcdn_set_debug(s.ctx, dbg)
        try:
            s.set_launch(mode, ctas, args.heavy)
        except pk.PCDNError as e:
            print(json.dumps({"P": P, "mode": mode, "error": str(e)}), flush=True)
            continue
        s.reset()
        s.solve(P, seed=prob.seed, max_outer=1)   # warm
        s.reset()
        if args.profile:
            pk.pcdn_set_profile(s.ctx, 1)
        r = s.solve(P, seed=prob.seed, max_outer=args.outer)
        cyc, used = pk.pcdn_phase_cycles(s.ctx)
        if args.profile:
            pk.pcdn_set_profile(s.ctx, 0)
        steps = r["steps"]
        kms = r["t_step_kernel_ms"]
        gbs = r["alg_bytes"] / (kms / 1e3) / 1e9
        out = {"cfg": args.cfg, "P": P, "debug": dbg, "mode_req": mode, "ctas": ctas, "mode_used": used, "heavy_len": args.heavy, "outer": r["outer_iters"],
               "steps": steps, "step_us": 1e3 * kms / steps, "kernel_ms_per_outer": kms / max(1, r["outer_iters"]),
               "gpu_ms_per_outer": r["t_gpu_ms"] / max(1, r["outer_iters"]),
               "alg_bytes_per_step": r["alg_bytes"] / steps, "kernel_alg_GBs": gbs, "frac_measured_hbm": gbs / peak,
               "nnz_per_step": r["nnz_processed"] / steps, "touched_per_step": r["touched_total"] / steps,
               "F": r["F"], "launches": r["kernel_launches"]}
        if args.profile:
            out["phase_cycles"] = (cyc / steps).round().tolist()
        print(json.dumps(out), flush=True)
