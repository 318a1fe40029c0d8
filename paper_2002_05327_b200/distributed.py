"""RHS-parallel execution over ranks (one process per GPU).

SURVEY §8(e): right-hand sides are independent through the whole DDM and
GMRES pipeline, so the multi-GPU form of the hot path is replicas: every
rank factors the same subdomain operators (replicated, no communication),
solves a contiguous shard of the RHS batch, and the shards are gathered once
at the end.  There is no collective in the data path; `torch.distributed`
(NCCL on GPUs, gloo in the CPU tests) only gathers results and reduces the
per-rank timings (max over ranks).
"""

from __future__ import annotations


def rhs_shard(nrhs: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous [start, stop) of `nrhs` right-hand sides for `rank`."""
    base, extra = divmod(nrhs, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def solve_sharded(f, solve_fn, group=None):
    """Apply `solve_fn` to this rank's shard of `f` ([R, ...] tensor) and
    return the full [R, ...] result on every rank (one all_gather)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    R = f.shape[0]
    lo, hi = rhs_shard(R, rank, world)
    # an empty shard (R < world) still joins the all_gather below; solve_fn
    # must accept a [0, ...] batch (diagonal_sweep_solve returns an empty field)
    out = solve_fn(f[lo:hi])
    width = max(rhs_shard(R, r, world)[1] - rhs_shard(R, r, world)[0] for r in range(world))
    pad = torch.zeros((width,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    pad[: hi - lo] = out
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][: rhs_shard(R, r, world)[1] - rhs_shard(R, r, world)[0]]
                      for r in range(world)], 0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The max of a per-rank scalar (e.g. a CUDA-event time) over ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
