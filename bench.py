#!/usr/bin/env python
"""PCDN (arXiv:1306.4080) hot-path benchmark on B200 -- the driver's bench contract.

A "step" is one full PCDN solve of the workload from w0 = 0 (Alg.3) to the
Eq.14 relative objective gap eps = 1e-3: every row of SURVEY.md 8(a)
(partition a0, g/h/d a1-a2, d'x a3, Armijo a4, commit a5, outer refresh + stop test a6)
runs inside it.  Default workload = config 5, the largest single-GPU configuration of
BASELINE.json (BASELINE.json's metric names no config): L1-logistic regression, kdda-shaped
2,000,000 x 20,000,000, Zipf(1.05) column popularity, 40 nonzeros per row (80M), P=4096, seed 4,
solved from w0 = 0 to the Eq.14 gap 1e-3 against the committed F* (tests/golden/fstar.json).

value  = bundle nonzeros processed per second (sum over steps of sum_{j in B} nnz(x^j)),
         whole job (all ranks), inputs resident in HBM, device time from CUDA events.
e2e    = the same metric through pcdn_train_host() with pinned HOST buffers (H2D of the
         inputs and D2H of w inside the timed region).
--impl reference times the CPU oracle (oracle/, fp64, 1 thread) on the same workload: each of its
steps is a bounded sample (the first bundle steps of outer iteration 0 from w0 = 0, sized so the
whole --steps K --warmup W run takes a few minutes), reported in the same unit (nnz/s).

Multi-GPU: the path does not shard; under torchrun
every rank solves its own replica; value = all ranks' nonzeros / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCDN time to rel. obj gap 1e-3; nnz/s and HBM GB/s vs 8 TB/s roofline"
NOMINAL_HBM_GBS = 8000.0


def load_json(path, default=None):
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return default


def peaks():
    mp = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    if mp and "hbm_gbs" in mp:
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fstar_for(cfg, loss):
    g = load_json(os.path.join(ROOT, "tests", "golden", "fstar.json"), {})
    key = f"cfg{cfg}_{'lr' if loss == 0 else 'svm'}"
    if key not in g:
        raise SystemExit(f"no F* for {key} in tests/golden/fstar.json (run scripts/make_fstar.py)")
    return float(g[key]["F_star"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def aggregate_over_ranks(t_ms, totals, dist=None, device="cpu"):
    """Whole-job numbers of a replicas-only run: the timed region of the job is the
    slowest rank's (max over ranks), work counters add up over ranks.  Without a process group
    (N=1) the inputs are returned as they are."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(t_ms), {k: float(v) for k, v in totals.items()}
    tt = torch.tensor([float(t_ms)], dtype=torch.float64, device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    keys = sorted(totals)
    vv = torch.tensor([float(totals[k]) for k in keys], dtype=torch.float64, device=device)
    dist.all_reduce(vv, op=dist.ReduceOp.SUM)
    return float(tt.item()), {k: float(x) for k, x in zip(keys, vv.tolist())}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def pin_one_core():
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return 1


def oracle_sample(o, prob, nsteps):
    """The first `nsteps` bundle steps of outer iteration 0 from w0 = 0 (Alg.3 as the oracle runs
    it): (nonzeros processed, seconds inside the bundle steps, steps).  The call's setup (the
    partition pi_0 of all n features, state arrays) is outside the timed steps."""
    r = o.solve(prob.P, seed=prob.seed, max_outer=1, trace_cap=0, max_steps=int(nsteps))
    return r["nnz"], r["t_steps"], r["steps"]


def calibrate_oracle(o, prob, target_s):
    """Bundle steps of a sample that takes about target_s seconds (from a short timed run)."""
    b = -(-prob.n // prob.P)
    probe = max(1, min(b, 50))
    _, sec, st = oracle_sample(o, prob, probe)
    per = sec / max(1, st)
    return int(max(1, min(b, target_s / max(per, 1e-9))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--loss", type=int, default=None)
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--P", type=int, default=None)
    ap.add_argument("--outer", type=int, default=0,
                    help="run exactly this many outer iterations per solve (no Eq.14 stop test; for configs "
                         "without a committed F*)")
    ap.add_argument("--mode", type=int, default=0, help="step-kernel launch mode (pcdn_set_launch)")
    ap.add_argument("--mu", type=float, default=0.0,
                    help="elastic-net weight (pcdn_set_elastic; NEXT #4): needs --outer (no stored F*)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    import synth
    ws, rank, local = dist_setup()
    if args.loss == 2:   # Lasso / elastic-net regression on the config's design matrix (Z26)
        prob = synth.regression(synth.config(args.config), noise=0.1, support=min(500, synth.config(args.config).n))
    else:
        prob = synth.config(args.config, loss=args.loss)
    if args.P:
        prob.P = args.P
    if (args.mu > 0 or args.loss == 2) and args.outer <= 0:
        raise SystemExit("--mu / --loss 2 need --outer N (F* is stored for the paper's two losses, mu = 0)")
    fstar = fstar_for(args.config, prob.loss) if args.outer <= 0 else None
    lossname = {0: "L1-logistic", 1: "L1-L2-loss-SVM", 2: "Lasso (squared loss, planted targets)"}[prob.loss]
    stop = f"Eq.14 gap {args.eps:g}" if args.outer <= 0 else f"{args.outer} outer iterations"
    if args.mu > 0:
        lossname += f" + elastic net mu={args.mu:g}"
    workload = (f"cfg{args.config}: {lossname} s={prob.s} x n={prob.n}, nnz={prob.nnz}, c={prob.c}, "
                f"P={prob.P}, seed={prob.seed}, solve w0=0 -> {stop}")
    config = {"workload": workload, "config_index": args.config, "s": prob.s, "n": prob.n, "nnz": prob.nnz,
              "P": prob.P, "c": prob.c, "loss": lossname, "eps": args.eps, "F_star": fstar,
              "l2": "flushed between timed solves (256 MiB write)", "parallelism": f"replicas x{ws}"}

    if args.impl == "reference":
        # the reference arm is the CPU oracle (tier rule): rank 0 only, 1 pinned core; each step a
        # bounded sample of the workload, the whole run sized to a few minutes
        if rank != 0:
            return 0
        import oracle
        cores = pin_one_core()
        o = oracle.Oracle(prob)
        budget = float(os.environ.get("PCDN_REF_BUDGET_S", "180"))
        nsteps = calibrate_oracle(o, prob, max(1.0, budget / max(1, args.steps + args.warmup)))
        for _ in range(args.warmup):
            oracle_sample(o, prob, nsteps)
        nnz, sec, bsteps = 0, 0.0, 0
        for _ in range(args.steps):
            a_, b_, c_ = oracle_sample(o, prob, nsteps)
            nnz, sec, bsteps = nnz + a_, sec + b_, bsteps + c_
        value = nnz / sec
        sample = (f"each step: the first {nsteps} bundle steps (of {-(-prob.n // prob.P)} per outer iteration) of "
                  f"outer iteration 0 from w0 = 0, oracle/ fp64 single thread")
        line = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
                "data": "synthetic (seeded generator synth/, SURVEY.md 8(d) recipe)", "config": config,
                "bundle_steps_per_s": bsteps / sec,
                "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": cores, "kind": "oracle", "sample": sample,
                                 "cpu": cpu_model()},
                "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import paper_1306_4080_b200 as pk
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        solver = pk.Solver(prob, device=dev, stream=stream)
    if fstar is not None:
        pk.pcdn_set_reference(solver.ctx, fstar)
    if args.mu > 0:
        solver.set_elastic(args.mu)
    if args.mode:
        solver.set_launch(args.mode)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    eps_run, max_outer = (args.eps, 1000) if args.outer <= 0 else (0.0, args.outer)

    def one_solve():
        pk.pcdn_reset(solver.ctx)
        st, inf = pk.pcdn_solve(solver.ctx, prob.P, eps_run, prob.seed, max_outer)
        if st != (pk.PCDN_OK if args.outer <= 0 else pk.PCDN_BUDGET):
            raise SystemExit(f"solve did not reach the gap: status {st}")
        return inf

    for _ in range(args.warmup):
        one_solve()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    infos = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            ev0[k].record(stream)
            infos.append(one_solve())
            ev1[k].record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    nnz = sum(i.nnz_processed for i in infos)
    steps_b = sum(i.steps for i in infos)
    alg_bytes = sum(i.alg_bytes for i in infos)
    t_kernel = sum(i.t_step_kernel_ms for i in infos)
    launches = sum(i.kernel_launches for i in infos)
    outer = infos[-1].outer_iters
    # step-kernel launches (one per outer iteration) for per-launch roofline numbers
    step_launches = sum(i.outer_iters for i in infos)
    t_ms, tot = aggregate_over_ranks(t_ms, {"nnz": nnz, "steps": steps_b, "alg_bytes": alg_bytes},
                                     dist if ws > 1 else None, dev)
    nnz_all, steps_all, bytes_all = tot["nnz"], tot["steps"], tot["alg_bytes"]

    # end-to-end through the public one-call API with pinned host buffers
    e2e = None
    if not args.no_e2e and fstar is not None:
        pin = {}
        # the CSC and the labels only: the one-call API builds the CSR on the device
        for name, dt in (("col_ptr", np.int64), ("row_idx", np.int32), ("val", np.float32), ("y", np.int8)):
            a = np.ascontiguousarray(getattr(prob, name), dtype=dt)
            t = torch.empty(a.shape, dtype=getattr(torch, np.dtype(dt).name), pin_memory=True)
            t.numpy()[...] = a
            pin[name] = t
        w_host = torch.empty(prob.n, dtype=torch.float64, pin_memory=True)
        h2d = sum(t.numel() * t.element_size() for t in pin.values())
        d2h = w_host.numel() * w_host.element_size()

        def e2e_once():
            return pk.pcdn_train_host(pin["col_ptr"].numpy(), pin["row_idx"].numpy(), pin["val"].numpy(), None, None,
                                      None, pin["y"].numpy(), prob.c, prob.loss, prob.P, args.eps, fstar, prob.seed,
                                      1000, stream=stream, w_out=w_host.numpy())

        e2e_once()
        torch.cuda.synchronize(dev)
        e_nnz, e_ms = 0, 0.0
        for k in range(max(1, min(args.steps, 3))):
            with torch.cuda.stream(stream):
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st, inf, _ = e2e_once()
            b.record(stream)
            b.synchronize()
            e_ms += a.elapsed_time(b)
            e_nnz += inf.nnz_processed
        e_ms, e_tot = aggregate_over_ranks(e_ms, {"nnz": e_nnz}, dist if ws > 1 else None, dev)
        e2e = {"value": e_tot["nnz"] / (e_ms / 1e3), "unit": "nnz/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms / max(1, min(args.steps, 3)),
               "api": "pcdn_train_host (pinned host CSC + labels; the CSR built on the device; includes "
                      "create/validate/solve/copy-back)"}

    peak, peak_src = peaks()
    per_launch_bytes = alg_bytes / max(1, step_launches)
    per_launch_ms = t_kernel / max(1, step_launches)
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
    mode_used = pk.pcdn_phase_cycles(solver.ctx)[1]
    kname = {1: "k_step_sparse<ClusterSync>", 2: "k_step_sparse<GridSync>", 3: "k_step_res", 4: "k_step_dense",
             5: "k_step<GridSync>"}.get(mode_used, "k_step")
    # DRAM bytes per launch of this kernel, this config/loss/P, from the ncu pass of this round
    # (scripts/traffic_from_ncu.py writes profiles/traffic.json from the capture; null if absent)
    tkey = f"cfg{args.config}_loss{prob.loss}_P{prob.P}_{kname}"
    tent = load_json(os.path.join(ROOT, "profiles", "traffic.json"), {}).get(tkey, {})
    traffic = tent.get("dram_bytes_per_launch")
    launch_desc = ("persistent, one launch per solve: figures per outer iteration" if kname == "k_step_dense"
                   else "persistent, one launch per outer iteration")
    roof = {"bound": "hbm", "kernel": f"pcdn::{kname} ({launch_desc})",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": tent.get("source"), "alg_bytes_per_launch": per_launch_bytes,
            "launch_ms": per_launch_ms, "peak_source": peak_src,
            "share_of_step": t_kernel / t_ms if t_ms else None,
            "frac_of_nominal_8TBs": achieved / NOMINAL_HBM_GBS,
            "alg_model": "SURVEY.md 8(d): 16 B per bundle nonzero + 16 B per touched sample + 28 B per position"}
    if kname == "k_step_dense":
        # a fully dense problem needs no row indices and keeps the per-sample state on chip: the bytes
        # it must move are the fp32 values (4 B per bundle nonzero) plus the same per-sample/position
        # terms -- the 8(d) model counts 12 B per nonzero this layout does not move
        min_bytes = (alg_bytes - 12 * nnz) / max(1, step_launches)
        roof["dense_min_bytes_per_launch"] = min_bytes
        roof["dense_min_frac"] = min_bytes / (per_launch_ms / 1e3) / 1e9 / peak

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        # the oracle as it stands, 1 pinned core, on a bounded sample (~15 s) of the same workload:
        # the first bundle steps of outer iteration 0 from w0 = 0 (every d_j != 0 there, so the
        # most expensive steps per nonzero); its time to the gap is extrapolated from its nnz rate
        # over the GPU run's nonzeros (every outer iteration processes every column once)
        import oracle
        cores = pin_one_core()
        o = oracle.Oracle(prob)
        nst = calibrate_oracle(o, prob, float(os.environ.get("PCDN_CPU_SAMPLE_S", "15")))
        c_nnz, c_sec, c_steps = oracle_sample(o, prob, nst)
        rate = c_nnz / c_sec
        per_solve_nnz = nnz / max(1, args.steps)
        cpu = {"value": rate, "unit": "nnz/s", "cores": cores, "kind": "oracle",
               "sample": f"the first {c_steps} bundle steps of outer iteration 0 from w0 = 0 ({c_sec:.1f} s inside "
                         f"the steps; {c_nnz} bundle nonzeros)", "cpu": cpu_model(),
               "time_to_gap_s_extrapolated": per_solve_nnz / rate,
               "extrapolation": "GPU run's bundle nonzeros per solve / the sample's nnz rate (bundle steps only: "
                                "the per-outer partition build and objective refresh are not counted)"}

    if rank == 0:
        value = nnz_all / (t_ms / 1e3)
        line = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator synth/, SURVEY.md 8(d) recipe)", "config": config,
                "time_to_gap_s": t_ms / args.steps / 1e3, "outer_iters": outer,
                "bundle_steps_per_s": steps_all / (t_ms / 1e3),
                "step_us": 1e3 * t_kernel / max(1, steps_b), "step_launch_mode": pk.pcdn_phase_cycles(solver.ctx)[1],
                "hbm_gbs_alg_whole_step": bytes_all / (t_ms / 1e3) / 1e9,
                "frac_of_8TBs_whole_step": bytes_all / (t_ms / 1e3) / 1e9 / NOMINAL_HBM_GBS,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    solver.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
