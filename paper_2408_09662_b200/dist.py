"""Multi-process (one process per GPU) batch sharding.

The path shards trivially: instances are independent, so N ranks split the
batch with the reference's contiguous-chunk rule (``batchrt._chunk_bounds``,
/root/reference/pkg/src/vecsym/batchrt.py:189-191) and never exchange data
while evaluating.  ``batch_eval_ranks`` is the torchrun counterpart of
``batch_eval(devices=[...])`` (the in-process sharder, ``vsb_eval_host_sharded``):
every rank evaluates its shard of one workspace on its own GPU through the C
ABI's sub-range entry point, then the output shards are exchanged once (the
final gather) so every rank's workspace holds the whole batch.  Works with
``nccl`` (shards staged through the rank's GPU) and ``gloo``.
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_bounds", "max_over_ranks", "batch_eval_ranks"]


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of `rank`'s contiguous shard: B*k//W (batchrt.py:189-191)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return batch * rank // world, batch * (rank + 1) // world


def _group_info(group):
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return None, 1, 0
    return dist.get_backend(group), dist.get_world_size(group), dist.get_rank(group)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """MAX all-reduce of a scalar (the contract's max-over-ranks timing)."""
    import torch
    import torch.distributed as dist

    _, world, _ = _group_info(group)
    if world == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def batch_eval_ranks(tape, ws, *, device: int | None = None, group=None, plan_options=None, evaluate=None):
    """Evaluate workspace ``ws`` sharded over the ranks of ``group``; returns ``ws.outputs``.

    Rank r runs elements ``shard_bounds(B, world, r)`` on CUDA device ``device``
    (default: the rank's current device) with the plan's host-path entry point
    (pinned host buffers -> its GPU -> host), then one all-gather per output moves
    every shard to every rank.  ``evaluate(tape, ws, lo, hi)`` replaces the GPU call
    (the CPU multi-process tests inject the oracle there).
    """
    import torch
    import torch.distributed as dist

    from .batchrt import _plan_for
    from .tape import as_tape

    tape = as_tape(tape)
    if not ws.matches(tape):
        raise ValueError("workspace/tape mismatch")
    backend, world, rank = _group_info(group)
    B = ws.batch_size
    lo, hi = shard_bounds(B, world, rank)
    if evaluate is not None:
        evaluate(tape, ws, lo, hi)
    elif hi > lo:
        dev = torch.cuda.current_device() if device is None else int(device)
        plan = _plan_for(tape, ws, plan_options)
        plan.eval_host(ws._in_buf.ctypes.data, ws._in_off, ws._out_buf.ctypes.data, ws._out_off, lo, hi, dev)
    if world == 1:
        return ws.outputs
    # final gather: shards padded to the largest, one all-gather per output
    spans = [shard_bounds(B, world, r) for r in range(world)]
    rows = max(h - l for l, h in spans)
    on_gpu = backend == "nccl"
    tdev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device)) if on_gpu else "cpu"
    for j, nz in enumerate(tape.nnz_out):
        if nz == 0:
            continue
        mine = torch.zeros((rows, nz), dtype=torch.float64 if ws.dtype == np.float64 else torch.float32, device=tdev)
        mine[: hi - lo] = torch.from_numpy(ws.output_matrix(j)[lo:hi])
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        out = ws.output_matrix(j)
        for r, (l, h) in enumerate(spans):
            if r != rank and h > l:
                out[l:h] = parts[r][: h - l].cpu().numpy()
    return ws.outputs
