"""Sample-sharded PCDN: each rank owns a row shard, w and the
partition stream are replicated, and one bundle step is the C-ABI's four phases with two
cross-rank sums between them (include/pcdn.h, "Sample-sharded step").  The sums are taken in rank
order from an all-gather, so every rank gets bit-identical g/h and line-search totals and takes
the identical decision (Eq.6).  Argument marshalling and the collectives only: every arithmetic
step of the path runs in libpcdn.so.

Usage (one process per GPU, torch.distributed initialised; world = 1 needs no process group):
    shard = synth.shard_rows(prob, rank, world)
    ss = ShardedSolver(shard, group=dist.group.WORLD if world > 1 else None)
    r = ss.solve(P, seed=..., max_outer=...)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import PCDN_BUDGET, PCDN_ERR_NUMERIC, PCDN_OK, PCDNError, Solver, check, lib, pcdn_permutation
from . import _ptr

W = 6   # candidates per line-search window (pcdn_shard_line_search)


def pcdn_shard_gh(ctx, bundle, P, gh_out):
    return check(ctx, lib().pcdn_shard_gh(ctx, _ptr(bundle), int(P), _ptr(gh_out)))


def pcdn_shard_direction(ctx, bundle, P, gh):
    return check(ctx, lib().pcdn_shard_direction(ctx, _ptr(bundle), int(P), _ptr(gh)))


def pcdn_shard_line_search(ctx, bundle, P, q0, first, with_l1, out):
    return check(ctx, lib().pcdn_shard_line_search(ctx, _ptr(bundle), int(P), int(q0), int(first), int(with_l1),
                                                   _ptr(out)))


def pcdn_shard_commit(ctx, bundle, P, alpha):
    return check(ctx, lib().pcdn_shard_commit(ctx, _ptr(bundle), int(P), float(alpha)))


def pcdn_shard_loss(ctx):
    v = C.c_double()
    check(ctx, lib().pcdn_shard_loss(ctx, C.byref(v)))
    return v.value


def rank_order_sum(t, group=None):
    """Sum of `t` over the ranks of `group`, added in rank order (identical bits on every rank).
    CPU tensors for gloo, device tensors for NCCL; world 1 (group None) returns t."""
    if group is None:
        return t
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    src = t if dist.get_backend(group) == "nccl" else t.cpu()
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    return acc.to(t.device)


class ShardedSolver:
    """One rank's share of a sample-sharded PCDN solve (the shard's rows; global n)."""

    def __init__(self, shard, group=None, **kw):
        import torch
        self.torch = torch
        self.group = group
        if group is None:
            self.rank = 0
        else:
            import torch.distributed as dist
            self.rank = dist.get_rank(group)
        self.sol = Solver(shard, **kw)
        self.ctx, self.n, self.c = self.sol.ctx, self.sol.n, self.sol.c
        self.mu = 0.0
        self.beta, self.sigma, self.qmax = 0.5, 0.01, 50
        dev = self.sol.device
        self.gh = torch.zeros(2 * self.n, dtype=torch.float64, device=dev)
        self.out = torch.zeros(2 * W + 1, dtype=torch.float64, device=dev)
        self.F = self.objective()

    def set_elastic(self, mu):
        self.sol.set_elastic(mu)
        self.mu = float(mu)
        self.F = self.objective()

    def objective(self):
        """Eq.1: the ranks' local losses summed in rank order, plus the separable terms of w."""
        w = self.sol.w().cpu().numpy()
        loss = rank_order_sum(self.torch.tensor([pcdn_shard_loss(self.ctx)], dtype=self.torch.float64),
                              self.group)
        return float(loss[0]) + float(np.sum(np.abs(w))) + 0.5 * self.mu * float(np.dot(w, w))

    def step(self, bundle):
        """One bundle step; returns (q, alpha, lhs) -- q = -1 for a null step (reading Z10)."""
        P = int(bundle.numel())
        gh = self.gh[:2 * P]
        pcdn_shard_gh(self.ctx, bundle, P, gh)
        gh.copy_(rank_order_sum(gh, self.group))
        pcdn_shard_direction(self.ctx, bundle, P, gh)
        q0, first, qacc, alpha_acc, lhs_acc = 0, 1, -1, 0.0, 0.0
        while q0 <= self.qmax:
            pcdn_shard_line_search(self.ctx, bundle, P, q0, first, self.rank == 0, self.out)
            tot = rank_order_sum(self.out, self.group).cpu().numpy()
            Delta = tot[2 * W]
            al = self.beta ** 0
            for _ in range(q0):
                al *= self.beta
            for q in range(W):
                lhs = tot[W + q] + self.c * tot[q]
                if not (np.isfinite(lhs) and np.isfinite(Delta)):
                    raise PCDNError(PCDN_ERR_NUMERIC, "non-finite line-search quantities")
                if q0 + q > self.qmax:
                    break
                if lhs <= self.sigma * al * Delta:
                    qacc, alpha_acc, lhs_acc = q0 + q, al, lhs
                    break
                al *= self.beta
            if qacc >= 0:
                break
            q0 += W
            first = 0
        pcdn_shard_commit(self.ctx, bundle, P, alpha_acc)
        if qacc >= 0:
            self.F += lhs_acc
        return qacc, alpha_acc, lhs_acc

    def solve(self, P, seed=0, max_outer=10, eps=0.0, fstar=None, trace=False):
        """Alg.3 with the Eq.14 stop test at outer boundaries (F refreshed there, reading Z23)."""
        torch = self.torch
        perm = torch.empty(self.n, dtype=torch.int32, device=self.sol.device)
        qs, Fs, steps, status, outer = [], [], 0, PCDN_BUDGET, 0
        for k in range(max_outer):
            pcdn_permutation(self.ctx, seed, k, perm)
            for t0 in range(0, self.n, P):
                q, _, _ = self.step(perm[t0:min(t0 + P, self.n)])
                steps += 1
                if trace:
                    qs.append(q)
                    Fs.append(self.F)
            self.F = self.objective()
            outer = k + 1
            if eps > 0 and fstar is not None and (self.F - fstar) / fstar <= eps:
                status = PCDN_OK
                break
        return dict(rc=status, F=self.F, steps=steps, outer_iters=outer, q_trace=np.array(qs, dtype=np.int32),
                    F_trace=np.array(Fs))

    def w(self):
        return self.sol.w()

    def close(self):
        self.sol.close()
