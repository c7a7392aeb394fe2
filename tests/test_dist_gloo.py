"""World-size-2 multi-process test of the batch-sharding plumbing on CPU
(gloo).  Each rank evaluates its contiguous shard (with the CPU oracle as the
per-rank evaluator, since this container has no GPU), the shards are
gathered to rank 0 and must equal a single-process evaluation bit for bit;
the timing reduction must return the max over ranks."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_09662_b200.dist import gather_rows, max_over_ranks, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, q):
    import sys

    sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    import oracle
    import workloads

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tape = workloads.load_tape("cartpole_rk4")
        ins = workloads.make_inputs("cartpole_rk4", batch, seed=42)
        lo, hi = shard_bounds(batch, world, rank)
        (out,) = oracle.batch_eval(tape, [v[lo:hi] for v in ins])
        full = gather_rows(out, batch)
        t = max_over_ranks(float(rank + 1) * 1.5)
        dist.barrier()
        q.put((rank, lo, hi, None if full is None else full.tobytes(), t))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_batch():
    for B in (1, 7, 103, 4096):
        for W in (1, 2, 3, 8):
            spans = [shard_bounds(B, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_two_rank_shard_gather_and_max_timing():
    import oracle
    import workloads

    world, batch = 2, 1001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [(0, 500), (500, 1001)]
    assert all(r[4] == 3.0 for r in res)  # max over ranks of (rank+1)*1.5
    tape = workloads.load_tape("cartpole_rk4")
    ins = workloads.make_inputs("cartpole_rk4", batch, seed=42)
    (ref,) = oracle.batch_eval(tape, ins)
    full = np.frombuffer(res[0][3], dtype=np.float64).reshape(ref.shape)
    assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))
    assert res[1][3] is None
