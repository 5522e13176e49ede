"""Multi-GPU plumbing for the CIRR stage.

The path shards by independent objects: whole GEPs (config 2's batch, or the
weak-scaling bench where each rank solves its own GEP).  There is no
data-path collective; torch.distributed is used only for the barrier and the
max-over-ranks timing reduction.  (Sharding one GEP's (contour x node)
pencils across GPUs would need one reduction of the moment block per
contour -- SURVEY.md 8(e) -- and is not built: BASELINE targets one GPU.)
"""

from __future__ import annotations


def shard(n_items: int, rank: int, world: int) -> list[int]:
    """Contiguous block partition of item indices 0..n_items-1 over ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (identity when not initialised)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
