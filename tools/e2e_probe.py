"""End-to-end probe (GPU box): batch_eval wall time per call through pinned host
buffers, and raw pinned H2D/D2H bandwidth.  One JSON line.

    VSB_HOST_PIECE_BYTES=1048576 python tools/e2e_probe.py --workload srbm_mpc --batch 4096
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="srbm_mpc")
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--calls", type=int, default=20)
    args = ap.parse_args()
    import torch

    import paper_2408_09662_b200 as vsb
    import workloads

    tape = workloads.load_tape(args.workload)
    ws = vsb.BatchWorkspace(tape, args.batch)
    for i, v in enumerate(workloads.make_inputs(args.workload, args.batch, seed=1)):
        ws.set_input(i, v)
    t_warm = time.perf_counter()
    while time.perf_counter() - t_warm < 1.0:   # PCIe link warm-up (tools/h2d_probe2.py)
        vsb.batch_eval(tape, ws)
    t = []
    for _ in range(args.calls):
        t0 = time.perf_counter()
        vsb.batch_eval(tape, ws)
        t.append(time.perf_counter() - t0)
    nbytes = ws._in_buf.nbytes
    h = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
    d = torch.empty_like(h, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    h2d = 10 * nbytes / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    d2h = 10 * nbytes / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"workload": args.workload, "batch": args.batch,
                      "piece_bytes": os.environ.get("VSB_HOST_PIECE_BYTES", "default"),
                      "ms_median": 1e3 * float(np.median(t)), "ms_min": 1e3 * min(t),
                      "evals_per_s": args.batch / float(np.median(t)), "h2d_gbs": h2d, "d2h_gbs": d2h,
                      "in_bytes": nbytes, "out_bytes": ws._out_buf.nbytes,
                      "zc_out": os.environ.get("VSB_ZC_OUT", "default"),
                      "out_sha": __import__("hashlib").sha256(ws._out_buf.tobytes()).hexdigest()[:16]}))


if __name__ == "__main__":
    main()
