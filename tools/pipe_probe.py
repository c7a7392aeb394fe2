"""End-to-end throughput of BatchPipeline vs synchronous batch_eval (GPU box).

    python tools/pipe_probe.py srbm_mpc 4096 --depth 1 2 3 --steps 50

Every step copies its inputs from pinned host memory and its outputs back; `depth`
workspaces rotate (a workspace is resubmitted only after its ticket was waited for).
Prints one JSON line per configuration."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("batch", type=int)
    ap.add_argument("--depth", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    import paper_2408_09662_b200 as vsb
    import workloads

    tape = workloads.load_tape(args.workload)
    ins = workloads.make_inputs(args.workload, args.batch, seed=3)

    def ws_new():
        ws = vsb.BatchWorkspace(tape, args.batch)
        for i, v in enumerate(ins):
            ws.set_input(i, v)
        return ws

    ws0 = ws_new()
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:
        vsb.batch_eval(tape, ws0)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vsb.batch_eval(tape, ws0)
    sync = args.batch * args.steps / (time.perf_counter() - t0)
    print(json.dumps({"workload": args.workload, "batch": args.batch, "mode": "sync", "evals_s": sync}), flush=True)
    for depth in args.depth:
        wss = [ws_new() for _ in range(depth)]
        with vsb.BatchPipeline(tape, depth=depth) as pipe:
            def run(k_steps):
                tickets = []
                for k in range(k_steps):
                    if k >= depth:
                        pipe.wait(tickets[k - depth])
                    tickets.append(pipe.submit(wss[k % depth]))
                for t in tickets[max(0, k_steps - depth):]:
                    pipe.wait(t)
            run(10)
            t0 = time.perf_counter()
            run(args.steps)
            rate = args.batch * args.steps / (time.perf_counter() - t0)
        print(json.dumps({"workload": args.workload, "batch": args.batch, "mode": "pipe", "depth": depth,
                          "evals_s": rate, "vs_sync": rate / sync}), flush=True)


if __name__ == "__main__":
    main()
