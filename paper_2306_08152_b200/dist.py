"""Multi-start sharding across GPUs: plumbing only.

Starts are independent, so under the per-start policy ranks exchange nothing
during the sweeps.  Under the paper's batch policy (NEXT-1) the
ranks' shards form one batch: after every sweep the library calls a reducer
that sums three counts over the group (`batch_reducer`).  At the end of a run: NCCL allgather of the per-start 16-byte summaries, the argmin
kernel (qf_select_best_device) on the gathered table, and a broadcast of the
winner's gates from the rank that owns it.  One process per GPU, launched by
torchrun; torch.distributed provides the process group.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import BATCH_REDUCE_FN, qf_select_best_device


@dataclass
class Shard:
    """This rank's contiguous range of global starts.

    Weak scaling (`Shard(rank, world, S)`): every rank owns S starts,
    [r*S, (r+1)*S).  Strong scaling (`Shard.strong(total, world, rank)`): the
    job's `total` starts split by `shard_range` (sizes differ by <= 1).  The
    end-of-run allgather pads every rank's table to `S_max` records."""

    rank: int
    world: int
    S: int
    total: int | None = None  # strong scaling: the job's start count

    @classmethod
    def strong(cls, total: int, world: int, rank: int) -> "Shard":
        b, e = shard_range(total, world, rank)
        return cls(rank, world, e - b, total)

    def range_of(self, rank: int):
        if self.total is None:
            return rank * self.S, (rank + 1) * self.S
        return shard_range(self.total, self.world, rank)

    @property
    def start_begin(self) -> int:
        return self.range_of(self.rank)[0]

    @property
    def S_max(self) -> int:
        if self.total is None:
            return self.S
        return -(-self.total // self.world)

    def owner(self, global_index: int):
        """(rank, local index) owning a global start index."""
        g = int(global_index)
        for r in range(self.world):
            b, e = self.range_of(r)
            if b <= g < e:
                return r, g - b
        raise IndexError(global_index)


def shard_range(total: int, world: int, rank: int):
    """Strong-scaling split of `total` starts: contiguous, sizes differ by <= 1."""
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def exchange_best(shard: Shard, summ: torch.Tensor, gates_out: torch.Tensor, stream=None,
                  select=None):
    """End-of-run exchange.  summ: uint8 tensor of S x 16-byte qf_summary;
    gates_out: (S, var) float64.  Returns (best global index, winner gates)
    on every rank.  `select(gathered, count) -> int` defaults to the argmin
    kernel on the device.  Ranks with fewer than S_max starts pad their table
    with NaN-Delta records (a NaN never wins the argmin)."""
    rec = 16
    pad = shard.S_max - shard.S
    if pad:
        filler = torch.zeros(pad * rec, dtype=torch.uint8, device=summ.device)
        filler.view(torch.float64)[0::2] = float("nan")
        summ = torch.cat([summ[: shard.S * rec], filler])
    gathered = torch.empty(shard.world * shard.S_max * rec, dtype=torch.uint8, device=summ.device)
    dist.all_gather_into_tensor(gathered, summ.contiguous())
    count = shard.world * shard.S_max
    if select is None:
        best_t = torch.empty(1, dtype=torch.int64, device=summ.device)
        qf_select_best_device(gathered, count, best_t, stream)
        best_p = int(best_t.item())
    else:
        best_p = int(select(gathered, count))
    r, local = divmod(best_p, shard.S_max)  # padded layout -> (rank, local)
    owner = r
    best = shard.range_of(r)[0] + local
    if shard.rank == owner:
        buf = gates_out[local].contiguous().clone()
    else:
        buf = torch.empty(gates_out.shape[1], dtype=gates_out.dtype, device=gates_out.device)
    dist.broadcast(buf, src=owner)
    return best, buf


def reduce_counts(counts, group=None, device=None):
    """Sum a small int64 vector over the process group (in place on a host
    tensor); NCCL groups reduce a device copy."""
    t = torch.as_tensor(counts, dtype=torch.int64)
    backend = dist.get_backend(group)
    if backend == "nccl":
        d = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(d, op=dist.ReduceOp.SUM, group=group)
        t.copy_(d.cpu())
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def batch_reducer(group=None, device=None):
    """A qf_batch_reduce_fn (qf.h) for qf_params.batch_reduce that sums the
    per-sweep batch counts over `group`.  Keep the returned object alive for
    the duration of the call."""

    def _fn(user, counts, n):
        try:
            vals = [int(counts[i]) for i in range(n)]
            out = reduce_counts(vals, group, device)
            for i in range(n):
                counts[i] = int(out[i])
            return 0
        except Exception:  # reported to the caller as QF_E_NCCL
            return 1

    return BATCH_REDUCE_FN(_fn)
