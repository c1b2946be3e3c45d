"""Multi-GPU path on CPU (gloo, world_size 2).  The PCDN hot path does not shard (DESIGN.md 9:
replicas only): under torchrun every rank solves its own replica of the same seeded workload and
bench.py reports all ranks' work over the slowest rank's time.  These tests cover that host-side
logic without a GPU: the max/sum aggregation and that every rank builds the identical replica."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import bench
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t_ms = [12.5, 20.0][rank]
        totals = {"nnz": [1000, 3000][rank], "steps": [7, 9][rank]}
        t, tot = bench.aggregate_over_ranks(t_ms, totals, dist, "cpu")
        digest = synth.config(1).digest()
        out = [None] * world
        dist.all_gather_object(out, digest)
        q.put((rank, t, tot, out))
    finally:
        dist.destroy_process_group()


def test_replicas_aggregate_and_identical_workload():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, tot, digests in res:
        assert t == 20.0                                  # max over ranks
        assert tot == {"nnz": 4000.0, "steps": 16.0}      # sums over ranks
        assert len(set(digests)) == 1                     # every rank: the same seeded replica


def test_aggregate_single_process():
    import bench
    t, tot = bench.aggregate_over_ranks(3.0, {"nnz": 5}, None)
    assert t == 3.0 and tot == {"nnz": 5.0}


def _sum_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1306_4080_b200.sharded import rank_order_sum
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(100 + rank)
        t = torch.randn(64, dtype=torch.float64, generator=g) * 10 ** torch.randint(-8, 8, (64,), generator=g)
        s = rank_order_sum(t, dist.group.WORLD)
        q.put((rank, t.numpy(), s.numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_rank_order_sum():
    """The sample-sharded step's cross-rank sums (gloo, world 2): every rank gets the identical
    bits, equal to the parts added in rank order (so every rank takes the same decision)."""
    import numpy as np
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_sum_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = res[0][1] + res[1][1]
    assert np.array_equal(res[0][2], want) and np.array_equal(res[1][2], want)
