"""Multi-GPU element sharding.

The volume term of element e reads only element e's data and D
(no cross-element index in volume.f90:11-160), so the
path shards into contiguous element ranges with NO collective on the data
path. One process per GPU; the only collective is a final 16-double
checksum (per-field sum and max-abs of rhsq) reduced over NCCL (gloo in
the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(ne: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous element range [start, stop) of ``rank``: sizes differ by
    at most one element; ranks cover [0, ne) exactly once, in order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if ne < 0:
        raise ValueError("ne must be non-negative")
    return ne * rank // world, ne * (rank + 1) // world


def local_checksum(rhsq: torch.Tensor) -> torch.Tensor:
    """[16] float64: per-field sum (8) then per-field max |.| (8) of an
    element-batched rhsq (Ne, 8, k, j, i)."""
    x = rhsq.to(torch.float64)
    if x.shape[0] == 0:
        return torch.zeros(16, dtype=torch.float64, device=rhsq.device)
    per = x.transpose(0, 1).reshape(8, -1)
    return torch.cat([per.sum(dim=1), per.abs().amax(dim=1)])


def global_checksum(rhsq: torch.Tensor, group=None) -> torch.Tensor:
    """All-reduced checksum: sums add, max-abs take the max. Without an
    initialised process group this is the local checksum."""
    c = local_checksum(rhsq)
    if not (dist.is_available() and dist.is_initialized()):
        return c
    sums, maxes = c[:8].clone(), c[8:].clone()
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(maxes, op=dist.ReduceOp.MAX, group=group)
    return torch.cat([sums, maxes])


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
