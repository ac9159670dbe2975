"""Multi-GPU partitioning: contiguous shards, one process per GPU, no
collective on the data path (every matrix is independent, nothing is
reduced).

    rank r of W owns rows [start, stop) = shard_range(n, r, W)

`run_sharded` is the one-call helper: each rank slices its shard of a
host (numpy) batch, runs it through the given per-rank solver, and —
only if asked — gathers the results to rank 0 with torch.distributed
(gather is a convenience for verification, never part of the metric).
"""

from __future__ import annotations

from typing import Callable, Optional


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced (sizes differ by at most one) row range."""
    if world <= 0 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad shard request n={n} rank={rank} world={world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def shard_sizes(n: int, world: int) -> list[int]:
    return [b - a for a, b in (shard_range(n, r, world) for r in range(world))]


def run_sharded(A, solve: Callable, rank: int, world: int, gather: bool = False,
                group: Optional[object] = None):
    """Solve this rank's contiguous shard of A; optionally gather to rank 0.

    `solve(A_shard) -> dict[str, np.ndarray]`.  Returns the local result, or
    on rank 0 with gather=True the row-ordered concatenation of all shards.
    """
    import numpy as np

    start, stop = shard_range(A.shape[0], rank, world)
    local = {k: v for k, v in solve(A[start:stop]).items() if v is not None}
    if not gather or world == 1:
        return local
    import torch.distributed as dist

    parts = [None] * world
    dist.all_gather_object(parts, {k: np.asarray(v) for k, v in local.items()}, group=group)
    if rank != 0:
        return local
    return {k: np.concatenate([p[k] for p in parts]) for k in local}
