#!/usr/bin/env python
"""Device-path timing of plans over workloads x batches x option grids (GPU box).

    python tools/sweep.py --workload srbm_mpc --batch 4096 65536 \
        --grid team=8,16 min_blocks=1,2 [--steps 10] [--check 16]

For every combination: inputs resident in HBM, L2 flushed (256 MiB write)
before each step outside the CUDA events, median of ``--steps`` steps after
3 warm-ups.  ``--check R`` compares R random rows with the CPU oracle.
One JSON line per configuration on stdout (plan statistics included).
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))


def parse_grid(items):
    keys, vals = [], []
    for it in items:
        k, v = it.split("=", 1)
        keys.append(k)
        vals.append([int(x) if x.lstrip("-").isdigit() else x for x in v.split(",")])
    return [dict(zip(keys, combo)) for combo in itertools.product(*vals)] if keys else [{}]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", nargs="+", required=True)
    ap.add_argument("--batch", type=int, nargs="+", default=[4096])
    ap.add_argument("--grid", nargs="*", default=[])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--check", type=int, default=0)
    ap.add_argument("--env", nargs="*", default=[], help="KEY=VALUE environment settings (before plan creation)")
    ap.add_argument("--compile-only", action="store_true",
                    help="NVRTC-compile the plans into the cubin cache and print their statistics (no GPU)")
    args = ap.parse_args()
    for kv in args.env:
        k, v = kv.split("=", 1)
        os.environ[k] = v

    import paper_2408_09662_b200 as vsb
    import workloads

    if args.compile_only:
        for name in args.workload:
            for opts in parse_grid(args.grid):
                info = vsb.Plan(workloads.load_tape(name), **opts).info
                print(json.dumps({"workload": name, "opts": opts, "env": args.env, "info": info}), flush=True)
        return

    import torch

    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for name in args.workload:
        tape = workloads.load_tape(name)
        for B in args.batch:
            ins = workloads.make_inputs(name, B, seed=3000)
            nin, nout = tape.nnz_in, tape.nnz_out
            in_off = np.concatenate([[0], np.cumsum(np.asarray(nin, dtype=np.int64) * B)])
            out_off = np.concatenate([[0], np.cumsum(np.asarray(nout, dtype=np.int64) * B)])
            d_in = torch.tensor(np.concatenate([v.ravel() for v in ins]), device=dev)
            d_out = torch.empty(int(out_off[-1]), dtype=torch.float64, device=dev)
            for opts in parse_grid(args.grid):
                rec = {"workload": name, "batch": B, "opts": opts, "env": args.env}
                try:
                    plan = vsb.Plan(tape, **opts)
                except Exception as e:  # noqa: BLE001 -- record and go on
                    rec["error"] = str(e)[:400]
                    print(json.dumps(rec), flush=True)
                    continue

                def step():
                    plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, 0, B, 0, stream.cuda_stream)

                try:
                    for _ in range(args.warmup):
                        flush.zero_()
                        step()
                    ms = []
                    for _ in range(args.steps):
                        flush.zero_()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        step()
                        b.record(stream)
                        b.synchronize()
                        ms.append(a.elapsed_time(b))
                except Exception as e:  # noqa: BLE001
                    rec["error"] = str(e)[:400]
                    print(json.dumps(rec), flush=True)
                    continue
                t = statistics.median(ms)
                info = plan.info
                rec.update({"ms": t, "ms_min": min(ms), "evals_s": B / (t / 1e3),
                            "io_gbs": 8 * (sum(nin) + sum(nout)) * B / (t / 1e3) / 1e9,
                            "info": {k: info[k] for k in ("team", "n_chunks", "phases", "xfers", "smem_slots",
                                                          "overflow_slots", "scratch_slots", "scratch_loads",
                                                          "max_regs", "max_local_bytes", "est_efficiency",
                                                          "code_bytes", "block", "groups", "cluster")}})
                if args.check:
                    import oracle

                    rows = np.random.default_rng(0).choice(B, size=min(B, args.check), replace=False)
                    ref = oracle.batch_eval(tape, [v[rows] for v in ins], n_threads=8)
                    got = d_out.cpu().numpy()
                    worst = 0.0
                    for j in range(tape.n_out):
                        g = got[out_off[j]:out_off[j + 1]].reshape(B, nout[j])[rows]
                        with np.errstate(invalid="ignore"):
                            e = np.abs(g - ref[j]) / np.maximum(np.abs(ref[j]), 1.0)
                        worst = max(worst, float(np.nanmax(e)) if e.size else 0.0)
                    rec["max_rel_err"] = worst
                print(json.dumps(rec), flush=True)
            del d_in, d_out


if __name__ == "__main__":
    main()
