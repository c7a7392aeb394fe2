#!/usr/bin/env python
"""Per-phase timeline of a team kernel chain (GPU box; diagnostic).

    python tools/phase_trace.py --workload srbm_mpc --batch 512 4096 > trace.json

Compiles the plan with VSB_PHASE_TRACE=1 (lane 0 of every warp of CTA 0 stores clock64()
when it reaches each phase barrier and when it leaves it), runs one warm-up and one traced
evaluation, reads ``vs_ptrace`` of every chunk through ``vsb_debug_read_global`` and prints
one JSON line per (batch, chunk): ``arrive[P][W]`` / ``depart[P][W]`` cycles relative to the
earliest warp start, plus the scheduler's per-warp phase loads (``load[P][W]``, cost units)
recomputed from the same plan's schedule statistics (VSB_SCHED_DEBUG goes to stderr).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="srbm_mpc")
    ap.add_argument("--batch", type=int, nargs="+", default=[512, 4096])
    ap.add_argument("--grid", nargs="*", default=[], help="plan options key=value")
    args = ap.parse_args()
    os.environ["VSB_PHASE_TRACE"] = "1"
    os.environ.setdefault("VSB_CACHE_DIR", "/tmp/vsb_trace_cache")

    import torch

    import paper_2408_09662_b200 as vsb
    from paper_2408_09662_b200 import _native
    import workloads

    opts = {}
    for kv in args.grid:
        k, v = kv.split("=", 1)
        opts[k] = int(v)
    tape = workloads.load_tape(args.workload)
    plan = vsb.Plan(tape, **opts)
    info = plan.info
    W = int(info["team"])
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    for B in args.batch:
        ins = workloads.make_inputs(args.workload, B, seed=3000)
        nin, nout = tape.nnz_in, tape.nnz_out
        in_off = np.concatenate([[0], np.cumsum(np.asarray(nin, dtype=np.int64) * B)])
        out_off = np.concatenate([[0], np.cumsum(np.asarray(nout, dtype=np.int64) * B)])
        d_in = torch.tensor(np.concatenate([v.ravel() for v in ins]), device=dev)
        d_out = torch.empty(int(out_off[-1]), dtype=torch.float64, device=dev)
        for _ in range(2):
            plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, 0, B, 0, stream.cuda_stream)
        torch.cuda.synchronize()
        for c in range(int(info["n_chunks"])):
            n = int(re.search(r"vs_ptrace\[(\d+)\]", plan.source(c)).group(1))
            P = (n - W) // (2 * W)
            buf = (ctypes.c_uint64 * n)()
            _native.check(_native.lib().vsb_debug_read_global(plan._h, c, b"vs_ptrace", 0, buf, 8 * n))
            a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
            start = a[2 * W * P:]
            t0 = int(start.min())
            tr = (a[:2 * W * P].reshape(P, W, 2) - t0)
            print(json.dumps({"workload": args.workload, "batch": B, "chunk": c, "W": W, "P": P, "opts": opts,
                              "start": (start - t0).tolist(), "arrive": tr[:, :, 0].tolist(),
                              "depart": tr[:, :, 1].tolist()}), flush=True)


if __name__ == "__main__":
    main()
