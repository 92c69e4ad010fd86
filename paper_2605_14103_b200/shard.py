"""Scenario sharding across GPUs (one process per GPU, no data-path collective).

Every scenario is an independent solve, so the batch is
split into contiguous index ranges, one per rank; each rank builds only its
own rows of the seeded batch (scenario i depends only on (seed, i)) and solves
them against its own replica of the plan. The only cross-rank operations are
outside the hot path: a barrier and the max-over-ranks reduction of the
timed interval, and an optional gather of per-scenario records.
"""

from __future__ import annotations

import os


def shard_range(total: int, rank: int, world: int) -> tuple:
    """[start, stop) of rank's contiguous share; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def dist_env() -> tuple:
    """(rank, local_rank, world) from torchrun's environment (1 process = 1 GPU)."""
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return rank, local, world


def max_over_ranks(value: float, device=None) -> float:
    """Max of a host float over all ranks (timing only; not on the data path)."""
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
