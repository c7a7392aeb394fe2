"""Closed-loop rollout throughput (GPU box): the paper's quadcopter use case
(10,000 environments, quad_step tape) as a device-resident
CUDA-graph loop vs the reference-style host loop on the CPU oracle.

    python tools/rollout_bench.py [--batch 10000] [--steps 100]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))


def main():
    import torch

    import oracle
    import workloads
    from paper_2408_09662_b200.rollout import Rollout

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="quad_step")
    ap.add_argument("--batch", type=int, default=10000)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--team", type=int, default=0)
    ap.add_argument("--hoist", choices=["auto", "on", "off"], default="auto")
    ap.add_argument("--fused", choices=["auto", "off"], default="auto")
    ap.add_argument("--shared-theta", action="store_true", help="one parameter row for every env (rollout_batch's broadcast)")
    ap.add_argument("--dedup", choices=["auto", "off"], default="auto")
    ap.add_argument("--no-record", action="store_true", help="final state only (roa_scan's mode)")
    args = ap.parse_args()
    tape = workloads.load_tape(args.workload)
    ins = workloads.make_inputs(args.workload, args.batch, seed=5)
    if args.shared_theta:
        ins = [ins[0]] + [np.repeat(v[:1], args.batch, axis=0) for v in ins[1:]]
    opts = {"team": args.team} if args.team else {}
    hoist = {"auto": None, "on": True, "off": False}[args.hoist]
    r = Rollout(tape, args.batch, args.steps, hoist=hoist, fused=None if args.fused == "auto" else False,
                dedup=None if args.dedup == "auto" else False, record=not args.no_record, **opts)
    r.set(torch.tensor(ins[0], device="cuda"), [torch.tensor(v, device="cuda") for v in ins[1:]])
    r.run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        r.run()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    gpu_rate = args.batch * args.steps / (ms / 1e3)
    # CPU: reference-style host loop (batch_eval + copy) with all host threads, bounded sample
    threads = len(os.sched_getaffinity(0))
    Bs = min(args.batch, 2000)
    ws = oracle.Workspace(tape, Bs)
    ws.set_inputs([v[:Bs] for v in ins])
    ws.run(threads)
    k_cpu = max(1, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(k_cpu):
        outs = ws.run(threads)
        ws.input_matrix(0)[:, :] = outs[0]
    cpu_s = time.perf_counter() - t0
    cpu_rate = Bs * k_cpu / cpu_s
    print(json.dumps({"workload": args.workload, "batch": args.batch, "steps": args.steps, "ms_per_rollout": ms,
                      "gpu_env_steps_per_s": gpu_rate, "cpu_env_steps_per_s": cpu_rate, "cpu_threads": threads,
                      "cpu_sample": f"{Bs} envs x {k_cpu} steps", "speedup": gpu_rate / cpu_rate,
                      "launches_per_rollout": r.launches_per_run, "plan": r.plan.info["team"],
                      "hoisted_rows": r.split.hoisted_rows if r.split is not None else 0, "fused": r.fused,
                      "distinct_param_rows": r.u_count or None, "shared_theta": args.shared_theta,
                      "record": not args.no_record}),
          flush=True)


if __name__ == "__main__":
    main()
