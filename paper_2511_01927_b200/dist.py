"""Multi-GPU plumbing for the CIRR stage.

The path shards by independent objects: whole GEPs (config 2's batch, or the
weak-scaling bench where each rank solves its own GEP), with no data-path
collective; torch.distributed then carries only the barrier and the
max-over-ranks timing reduction.  One GEP can also be split by quadrature node
(SURVEY.md 8(e)): ``solve_multi_node_sharded`` gives rank r the nodes r,
r + world, ... of every contour (its share of the factorisations and solves),
sums the partial moment blocks with one all-reduce per pass (NCCL over NVLink:
33 MB in config 4's first pass, 15 MB in the refinement passes) and lets every
rank run the same Rayleigh-Ritz on the identical sums.
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


def solve_multi_batch_sharded(pencils, contours, cfg=None, solver: str = "cirr", seeds=None, *, gather: bool = True,
                              solve_fn=None):
    """``solve_multi_batch`` over the ranks of the default process group (one
    rank per GPU): rank r solves the contiguous block ``shard(len(pencils), r,
    world)`` of the independent GEPs on its own device, with no data-path
    collective.  ``gather=True`` hands every rank all results in input order
    (one ``all_gather_object`` of the host-side results, after the solves);
    ``gather=False`` returns ``(indices, results)`` of this rank's block.
    ``contours`` / ``seeds`` as in solve_multi_batch (one list per pencil, or
    one list for all).  ``solve_fn`` replaces solve_multi_batch (same
    signature), e.g. to run the host logic without a GPU."""
    import torch.distributed as dist

    pencils = list(pencils)
    contours = list(contours)
    if contours and not isinstance(contours[0], (list, tuple)):
        contours = [contours] * len(pencils)
    if len(contours) != len(pencils):
        raise ValueError("need one contour list per pencil")
    seeds = [0] * len(pencils) if seeds is None else [int(x) for x in seeds]
    if len(seeds) != len(pencils):
        raise ValueError("need one seed per pencil")
    on = dist.is_available() and dist.is_initialized()
    rank, world = (dist.get_rank(), dist.get_world_size()) if on else (0, 1)
    mine = shard(len(pencils), rank, world)
    if solve_fn is None:
        from .solvers import solve_multi_batch as solve_fn
    res = solve_fn([pencils[i] for i in mine], [contours[i] for i in mine], cfg, solver,
                   [seeds[i] for i in mine]) if mine else []
    if not gather:
        return mine, res
    if world == 1:
        return list(res)
    parts = [None] * world
    dist.all_gather_object(parts, (mine, list(res)))
    out = [None] * len(pencils)
    for idx, rs in parts:
        for i, r in zip(idx, rs):
            out[i] = r
    return out


def _allreduce(group=None):
    """In-place all-reduce of a device tensor over the group: "sum" (complex tensors as their real
    view) or "min"."""
    import torch
    import torch.distributed as dist

    def run(t, op):
        v = torch.view_as_real(t) if t.is_complex() else t
        dist.all_reduce(v, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MIN, group=group)

    return run


def solve_multi_node_sharded(pencil, contours, cfg=None, solver: str = "cirr", seed: int = 0, *, group=None,
                             shard_ctx=None):
    """``solve_multi`` of ONE pencil over the ranks of ``group`` (one rank per
    GPU, every rank holding A and B): rank r factors and solves the quadrature
    nodes r, r + world, ... of every contour; after each solve pass the partial
    moment blocks are summed over the ranks (the path's one exchange step) and
    every rank continues with the same Rayleigh-Ritz, so all ranks return the
    same eigenpairs.  A singular shift found by any rank drops that contour on
    all of them (one min-reduction after the factorisation).  Per-rank
    ``stats`` count that rank's factorisations and solves.  ``shard_ctx``
    (a ``solvers.NodeShard``) replaces the torch.distributed group, e.g. for
    threads sharing one GPU in tests."""
    import torch.distributed as dist

    from . import solvers as S

    if shard_ctx is None:
        on = dist.is_available() and dist.is_initialized()
        rank, world = (dist.get_rank(group), dist.get_world_size(group)) if on else (0, 1)
        shard_ctx = S.NodeShard(rank, world, _allreduce(group))
    if cfg is not None and getattr(cfg, "conjugate_pairs", False) and shard_ctx.world > 1:
        raise S.ParameterError("the conjugate-pair variant and the node split are exclusive")
    prev = S.set_node_shard(shard_ctx)
    try:
        return S.solve_multi(pencil, contours, cfg, solver, seed)
    finally:
        S.set_node_shard(prev)
