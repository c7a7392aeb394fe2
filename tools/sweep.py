"""Parameter sweep of the device path (GPU box): ms/step and evals/s per
(workload, batch, plan options).  One JSON line per configuration.

    python tools/sweep.py --workload srbm_mpc --batch 4096 --grid block=32,64,128 chunk_ops=3000,6000
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))


def time_plan(plan, tape, inputs, B, steps, warmup, dev=0):
    import torch

    nin, nout = tape.nnz_in, tape.nnz_out
    in_off = np.concatenate([[0], np.cumsum(np.asarray(nin, dtype=np.int64) * B)])
    out_off = np.concatenate([[0], np.cumsum(np.asarray(nout, dtype=np.int64) * B)])
    d_in = torch.tensor(np.concatenate([v.ravel() for v in inputs]), device="cuda")
    d_out = torch.empty(int(out_off[-1]), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, 0, B, dev, s.cuda_stream)
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, 0, B, dev, s.cuda_stream)
        b.record(s)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms)), d_out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", nargs="+", default=["srbm_mpc"])
    ap.add_argument("--batch", nargs="+", type=int, default=[4096])
    ap.add_argument("--grid", nargs="*", default=[])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import paper_2408_09662_b200 as vsb
    import workloads

    keys, vals = [], []
    for g in args.grid:
        k, v = g.split("=")
        keys.append(k)
        vals.append([int(x) for x in v.split(",")])
    for name in args.workload:
        tape = workloads.load_tape(name)
        for B in args.batch:
            inputs = workloads.make_inputs(name, B, seed=0)
            for combo in itertools.product(*vals) if vals else [()]:
                opts = dict(zip(keys, combo))
                t0 = time.time()
                try:
                    plan = vsb.Plan(tape, **opts)
                    info = plan.info
                    ms, _ = time_plan(plan, tape, inputs, B, args.steps, args.warmup)
                except Exception as e:  # keep sweeping
                    print(json.dumps({"workload": name, "batch": B, "opts": opts, "error": str(e)[:500]}), flush=True)
                    continue
                print(json.dumps({
                    "workload": name, "batch": B, "opts": opts, "ms": ms, "evals_per_s": B / ms * 1e3,
                    "fp64_tops": tape.n_arith * B / ms / 1e9,
                    "io_gbs": 8 * (sum(tape.nnz_in) + sum(tape.nnz_out)) * B / ms / 1e6,
                    "plan": {k: info[k] for k in ("n_chunks", "block", "scratch_slots", "scratch_loads",
                                                  "scratch_stores", "max_regs", "max_local_bytes",
                                                  "stage_in", "stage_out", "compile_seconds")},
                    "wall_s": time.time() - t0}), flush=True)


if __name__ == "__main__":
    main()
