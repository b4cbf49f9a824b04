"""Multi-rank host logic of the end-of-run exchange on CPU
with the gloo backend, world size 2: shard ranges, allgather layout, argmin
with ties to the lowest global index, and the winner-gates broadcast."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2306_08152_b200 as qf
from paper_2306_08152_b200.dist import Shard, exchange_best, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, S, var, q, total=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # weak: S starts per rank; strong (bench.py --scaling strong): the
        # job's `total` starts split by shard_range, tables padded to S_max
        shard = Shard(rank, world, S) if total is None else Shard.strong(total, world, rank)
        S = shard.S
        summ = np.zeros(S, dtype=qf.SUMMARY_DTYPE)
        # deltas keyed by global start index; global 5 and 9 tie for the minimum
        g = np.arange(shard.start_begin, shard.start_begin + S)
        summ["delta"] = 0.5 + 0.01 * ((g * 7) % 11)
        summ["delta"][np.isin(g, [5, 9])] = 0.01
        summ["iters"] = g
        summ["verdict"] = 3
        t = torch.from_numpy(summ.view(np.uint8).copy())
        gates = torch.from_numpy(np.stack([np.full(var, float(x)) for x in g]))

        def host_select(gathered, count):
            return qf.qf_select_best_host(gathered.numpy().view(qf.SUMMARY_DTYPE)[:count])

        best, buf = exchange_best(shard, t, gates, select=host_select)
        q.put((rank, best, buf.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_exchange_best_gloo_world2():
    world, S, var = 2, 8, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, var, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, best, buf in out:
        assert best == 5  # tie between global 5 (rank 0) and 9 (rank 1) -> lowest index
        assert buf == [5.0] * var


@pytest.mark.parametrize("total", [13, 16])
def test_exchange_best_strong_gloo_world2(total):
    """bench.py's strong split: 13 starts over 2 ranks (7 + 6, rank 1 padded
    with a NaN record); global 5 (rank 0) and 9 (rank 1) tie -> 5."""
    world, var = 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 0, var, q, total))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, best, buf in out:
        assert best == 5
        assert buf == [5.0] * var
    s = Shard.strong(total, world, 1)
    assert s.start_begin == (total + 1) // 2 and s.S == total // 2 and s.S_max == (total + 1) // 2
    assert s.owner(total - 1) == (1, s.S - 1)


def test_shard_ranges():
    for total in (1, 7, 64, 1000, 8192):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    s = Shard(3, 8, 4096)
    assert s.start_begin == 3 * 4096 and s.owner(3 * 4096 + 17) == (3, 17)


def _batch_worker(rank, world, port, q):
    """The batch-policy reducer (qf_params.batch_reduce) called the way the
    library calls it: through the C function pointer, on int64 counts."""
    import ctypes

    from paper_2306_08152_b200.dist import batch_reducer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn = batch_reducer()
        # rank 0: one start converged, 3 running, 2 not plateaued; rank 1: none
        # converged, 5 running, 0 not plateaued
        local = [1, 2, 3] if rank == 0 else [0, 0, 5]
        arr = (ctypes.c_int64 * 3)(*local)
        rc = fn(None, ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64)), 3)
        q.put((rank, rc, list(arr)))
    finally:
        dist.destroy_process_group()


def test_batch_reducer_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank, rc, counts in out:
        assert rc == 0
        assert counts == [1, 2, 8]  # summed over the batch on every rank
