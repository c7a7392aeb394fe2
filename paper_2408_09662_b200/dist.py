"""Multi-process (one process per GPU) plumbing for batch sharding.

The path shards trivially: instances are independent, so N ranks split the
batch with the reference's contiguous-chunk rule (``batchrt._chunk_bounds``,
/root/reference/pkg/src/vecsym/batchrt.py:189-191) and never exchange data
while evaluating.  The only collectives are for timing (a barrier and a MAX
all-reduce) and an optional final gather of the shards' outputs to rank 0.
Works with any torch.distributed backend (``nccl`` on the GPU box, ``gloo``
in the CPU tests).
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_bounds", "max_over_ranks", "gather_rows"]


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of `rank`'s contiguous shard: B*k//W (batchrt.py:189-191)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return batch * rank // world, batch * (rank + 1) // world


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of a scalar (the contract's max-over-ranks timing)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: np.ndarray, batch: int, dst: int = 0):
    """Concatenate every rank's [rows, ...] shard on rank `dst` in rank order
    (the final device-to-host gather).  Returns the full array on `dst`, None
    elsewhere."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    parts = [None] * world if rank == dst else None
    dist.gather_object(np.ascontiguousarray(local), parts, dst=dst)
    if rank != dst:
        return None
    full = np.concatenate(parts, axis=0)
    if full.shape[0] != batch:
        raise RuntimeError(f"gathered {full.shape[0]} rows, expected {batch}")
    return full
