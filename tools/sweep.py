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
    tdt = torch.float32 if plan.np_dtype == np.float32 else torch.float64
    d_in = torch.tensor(np.concatenate([v.ravel() for v in inputs]), device="cuda", dtype=tdt)
    d_out = torch.empty(int(out_off[-1]), dtype=tdt, device="cuda")
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
    ap.add_argument("--dtype", default="float64")
    ap.add_argument("--check", type=int, default=0, help="compare N rows with the fp64 CPU oracle")
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
                    plan = vsb.Plan(tape, dtype=args.dtype, **opts)
                    info = plan.info
                    ms, d_out = time_plan(plan, tape, inputs, B, args.steps, args.warmup)
                except Exception as e:  # keep sweeping
                    print(json.dumps({"workload": name, "batch": B, "opts": opts, "error": str(e)[:500]}), flush=True)
                    continue
                check = None
                if args.check:
                    import oracle

                    rows = np.random.default_rng(1).choice(B, size=min(B, args.check), replace=False)
                    ref = oracle.batch_eval(tape, [v[rows] for v in inputs], n_threads=os.cpu_count() or 1)
                    out = d_out.double().cpu().numpy()
                    off = np.concatenate([[0], np.cumsum(np.asarray(tape.nnz_out) * B)])
                    errs = np.concatenate([
                        (np.abs(out[off[j]:off[j + 1]].reshape(B, -1)[rows] - ref[j])
                         / np.maximum(np.abs(ref[j]), 1.0)).ravel() for j in range(tape.n_out)])
                    errs = errs[np.isfinite(errs)]
                    check = {"rows": int(rows.size), "max_rel": float(errs.max()), "median_rel": float(np.median(errs)),
                             "p99_rel": float(np.quantile(errs, 0.99))}
                bpe = (4 if args.dtype == "float32" else 8) * (sum(tape.nnz_in) + sum(tape.nnz_out))
                print(json.dumps({
                    "workload": name, "batch": B, "dtype": args.dtype, "opts": opts, "ms": ms,
                    "evals_per_s": B / ms * 1e3, "fp64_tops": tape.n_arith * B / ms / 1e9,
                    "io_gbs": bpe * B / ms / 1e6, "check": check,
                    "plan": {k: info[k] for k in ("n_chunks", "block", "scratch_slots", "scratch_loads",
                                                  "scratch_stores", "max_regs", "max_local_bytes",
                                                  "stage_in", "stage_out", "compile_seconds", "team", "groups",
                                                  "cluster", "phases", "smem_slots", "overflow_slots", "xfers",
                                                  "remote_stores", "est_efficiency")},
                    "wall_s": time.time() - t0}), flush=True)


if __name__ == "__main__":
    main()
