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

from . import PCDN_BUDGET, PCDN_OK, Solver, check, lib, pcdn_permutation
from . import _ptr
from ._abi import pcdn_shard_decision

W = 6   # candidates per line-search window (pcdn_shard_line_search)


def pcdn_shard_gh(ctx, bundle, P, gh_out):
    return check(ctx, lib().pcdn_shard_gh(ctx, _ptr(bundle), int(P), _ptr(gh_out)))


def pcdn_shard_direction(ctx, bundle, P, gh):
    return check(ctx, lib().pcdn_shard_direction(ctx, _ptr(bundle), int(P), _ptr(gh)))


def pcdn_shard_line_search(ctx, bundle, P, q0, first, with_l1, out):
    return check(ctx, lib().pcdn_shard_line_search(ctx, _ptr(bundle), int(P), int(q0), int(first), int(with_l1),
                                                   _ptr(out)))


def pcdn_shard_decide(ctx, tot, q0):
    """The Eq.6 decision of one window from the rank-summed totals (on the device, with the
    context's Armijo constants); returns the pcdn_shard_decision."""
    d = pcdn_shard_decision()
    check(ctx, lib().pcdn_shard_decide(ctx, _ptr(tot), int(q0), C.byref(d)))
    return d


def pcdn_shard_commit(ctx, bundle, P):
    return check(ctx, lib().pcdn_shard_commit(ctx, _ptr(bundle), int(P)))


def pcdn_shard_loss(ctx, loss_out):
    return check(ctx, lib().pcdn_shard_loss(ctx, _ptr(loss_out)))


def pcdn_shard_objective(ctx, loss_sum):
    v = C.c_double()
    check(ctx, lib().pcdn_shard_objective(ctx, _ptr(loss_sum), C.byref(v)))
    return v.value


def rank_order_sum(t, group=None):
    """Sum of `t` over the ranks of `group`, added in rank order (identical bits on every rank): a
    deterministic all-reduce.  gloo takes CPU tensors, NCCL device tensors (the input's device);
    the result is on t's device.  World 1 (group None) returns t."""
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
    """One rank's share of a sample-sharded PCDN solve (the shard's rows; global n).  The Armijo
    constants (sigma, beta, gamma, q_max keywords) go to the context (pcdn_set_armijo); every
    decision is taken on the device from the rank-summed totals."""

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
        self.ctx, self.n = self.sol.ctx, self.sol.n
        dev = self.sol.device
        self.gh = torch.zeros(2 * self.n, dtype=torch.float64, device=dev)
        self.out = torch.zeros(2 * W + 1, dtype=torch.float64, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.F = self.objective()

    def set_elastic(self, mu):
        self.sol.set_elastic(mu)
        self.F = self.objective()

    def objective(self):
        """Eq.1 at an outer boundary: the ranks' local losses (device) summed in rank order, then F
        with the separable terms of w on the device (it becomes the maintained F)."""
        pcdn_shard_loss(self.ctx, self.loss)
        return pcdn_shard_objective(self.ctx, rank_order_sum(self.loss, self.group))

    def step(self, bundle):
        """One bundle step; returns the pcdn_shard_decision (q = -1: a null step, reading Z10)."""
        P = int(bundle.numel())
        gh = self.gh[:2 * P]
        pcdn_shard_gh(self.ctx, bundle, P, gh)
        gh.copy_(rank_order_sum(gh, self.group))
        pcdn_shard_direction(self.ctx, bundle, P, gh)
        q0, first = 0, 1
        while True:
            pcdn_shard_line_search(self.ctx, bundle, P, q0, first, self.rank == 0, self.out)
            dec = pcdn_shard_decide(self.ctx, rank_order_sum(self.out, self.group), q0)
            if dec.q >= 0 or not dec.next:
                break
            q0, first = q0 + W, 0
        pcdn_shard_commit(self.ctx, bundle, P)
        self.F = dec.F
        return dec

    def solve(self, P, seed=0, max_outer=10, eps=0.0, fstar=None, trace=False):
        """Alg.3 with the Eq.14 stop test at outer boundaries (F refreshed there, reading Z23).  The
        stop test compares the device-computed F with F* (the same value on every rank)."""
        torch = self.torch
        perm = torch.empty(self.n, dtype=torch.int32, device=self.sol.device)
        qs, Fs, steps, status, outer = [], [], 0, PCDN_BUDGET, 0
        for k in range(max_outer):
            pcdn_permutation(self.ctx, seed, k, perm)
            for t0 in range(0, self.n, P):
                dec = self.step(perm[t0:min(t0 + P, self.n)])
                steps += 1
                if trace:
                    qs.append(dec.q)
                    Fs.append(dec.F)
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
