"""Multi-GPU plumbing for the replicated hot path.

The path shards trivially: samples (displacement fields) and parts (independent meshes)
are independent units, so N ranks each process their own contiguous slice with no
data-path collective (weak scaling).  The only collective is the max-over-ranks of the
measured time (and an optional gather of per-sample totals), both host-side plumbing.
"""
from __future__ import annotations

import os


def world():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 without it)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_units: int, world_size: int, rank: int):
    """Contiguous, balanced [begin, end) slice of n_units for `rank` (sizes differ by <= 1)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad world_size / rank")
    base, rem = divmod(n_units, world_size)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a host float over all ranks (identity without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_totals(totals, device=None):
    """All-gather per-rank totals [S_r, K] into the global [sum S_r, K] (rank order)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return totals
    n = torch.tensor([totals.shape[0]], device=device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    m = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros((m,) + tuple(totals.shape[1:]), dtype=totals.dtype, device=device)
    pad[: totals.shape[0]] = totals
    out = [torch.zeros_like(pad) for _ in sizes]
    dist.all_gather(out, pad)
    return torch.cat([o[: int(s.item())] for o, s in zip(out, sizes)])
