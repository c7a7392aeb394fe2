"""World-size-2 multi-process test of ``dist.batch_eval_ranks`` on CPU (gloo).

Each rank evaluates its contiguous shard of one ``BatchWorkspace`` (the GPU
call is replaced by the CPU oracle on the same [lo, hi) range, since this
container has no GPU), the output shards are all-gathered, and every rank's
workspace must then equal a single-process evaluation bit for bit; the timing
reduction must return the max over ranks."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_09662_b200 import BatchWorkspace
from paper_2408_09662_b200.dist import batch_eval_ranks, max_over_ranks, shard_bounds


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
        ws = BatchWorkspace(tape, batch)
        for i, v in enumerate(ins):
            ws.set_input(i, v)
        seen = []

        def shard(tape_, ws_, lo_, hi_):   # the per-rank evaluator: oracle on [lo, hi)
            seen.append((lo_, hi_))
            outs = oracle.batch_eval(tape_, [ws_.input_matrix(i)[lo_:hi_] for i in range(tape_.n_in)])
            for j, o in enumerate(outs):
                ws_.output_matrix(j)[lo_:hi_] = o

        (full,) = batch_eval_ranks(tape, ws, evaluate=shard)
        lo, hi = seen[0]
        t = max_over_ranks(float(rank + 1) * 1.5)
        dist.barrier()
        q.put((rank, lo, hi, full.tobytes(), t))
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
    for r in res:   # every rank holds the whole batch after the final gather
        full = np.frombuffer(r[3], dtype=np.float64).reshape(ref.shape)
        assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))
