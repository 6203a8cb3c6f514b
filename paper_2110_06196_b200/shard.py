"""Walk-id sharding across ranks.

The global walk list is iteration-major (wid = it * n + node, §8(c) c13).
Rank r of G takes the contiguous wid range [floor(r W / G), floor((r+1) W / G))
and passes the range start as walk_id_base, so the concatenation of the ranks'
walk matrices equals the single-call matrix bit for bit.  No collective is on
the data path; torch.distributed only reduces timings / counters afterwards.
"""
from __future__ import annotations


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the global wid range owned by `rank` (contiguous, balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return total * rank // world, total * (rank + 1) // world


def weak_scaling_range(per_rank: int, rank: int, world: int) -> tuple[int, int]:
    """Weak scaling: the global list holds world * per_rank walks (per_rank per GPU);
    identical to shard_range(world * per_rank, rank, world)."""
    return shard_range(world * per_rank, rank, world)


def reduce_step_timing(local_ms: float, local_steps: float, world: int, device=None):
    """(max time over ranks, total steps over ranks) — the bench's whole-job figures."""
    if world == 1:
        return local_ms, local_steps
    import torch
    import torch.distributed as dist
    t = torch.tensor([local_ms], dtype=torch.float64, device=device)
    s = torch.tensor([local_steps], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return float(t.item()), float(s.item())
