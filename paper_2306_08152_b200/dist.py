"""Multi-start sharding across GPUs: plumbing only.

Starts are independent, so ranks exchange nothing during the sweeps.  At the
end of a run: NCCL allgather of the per-start 16-byte summaries, the argmin
kernel (qf_select_best_device) on the gathered table, and a broadcast of the
winner's gates from the rank that owns it.  One process per GPU, launched by
torchrun; torch.distributed provides the process group.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import qf_select_best_device


@dataclass
class Shard:
    """Weak-scaling shard: rank r owns global starts [r*S, (r+1)*S)."""

    rank: int
    world: int
    S: int

    @property
    def start_begin(self) -> int:
        return self.rank * self.S

    def owner(self, global_index: int):
        return divmod(int(global_index), self.S)


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
    kernel on the device."""
    gathered = torch.empty(shard.world * summ.numel(), dtype=torch.uint8, device=summ.device)
    dist.all_gather_into_tensor(gathered, summ)
    if select is None:
        best_t = torch.empty(1, dtype=torch.int64, device=summ.device)
        qf_select_best_device(gathered, shard.world * shard.S, best_t, stream)
        best = int(best_t.item())
    else:
        best = int(select(gathered, shard.world * shard.S))
    owner, local = shard.owner(best)
    if shard.rank == owner:
        buf = gates_out[local].contiguous().clone()
    else:
        buf = torch.empty(gates_out.shape[1], dtype=gates_out.dtype, device=gates_out.device)
    dist.broadcast(buf, src=owner)
    return best, buf
