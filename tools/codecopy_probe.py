"""Is the one-wave team chain slowed by many SMs fetching the SAME code at once?

srbm_mpc B=4096 runs 128 CTAs that execute identical instruction streams; 16 CTAs
take 0.305 ms, 128 take 0.416 ms.  Split the batch in two halves on two streams and
run them (a) with the same plan (same code addresses) and (b) with two plans whose
code differs only in schedule details (phase_cost 96 vs 95: same algorithm, different
instruction addresses).  If (b) is faster than (a), the CTAs contend on shared code
lines (L2 slices serving the same instruction lines to every SM).  Prints JSON lines.

Usage (GPU): python tools/codecopy_probe.py [--steps 30]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--alt", default="phase_cost=95")
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2408_09662_b200 as vsb
    import workloads

    name, B = "srbm_mpc", args.batch
    tape = workloads.load_tape(name)
    k, v = args.alt.split("=")
    pa = vsb.Plan(tape)
    pb = vsb.Plan(tape, **{k: int(v)})
    ins = workloads.make_inputs(name, B, seed=5)
    nin, nout = list(tape.nnz_in), list(tape.nnz_out)
    in_off = np.concatenate([[0], np.cumsum(np.asarray(nin, dtype=np.int64) * B)])
    out_off = np.concatenate([[0], np.cumsum(np.asarray(nout, dtype=np.int64) * B)])
    d_in = torch.tensor(np.concatenate([x.ravel() for x in ins]), device="cuda")
    outs = [torch.empty(int(out_off[-1]), dtype=torch.float64, device="cuda") for _ in range(3)]
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    h = B // 2

    def run(mode, out):
        if mode == "whole":
            pa.eval_device(d_in.data_ptr(), in_off, out.data_ptr(), out_off, 0, B, 0, s0.cuda_stream)
            return
        p2 = pa if mode == "halves_same_code" else pb
        pa.eval_device(d_in.data_ptr(), in_off, out.data_ptr(), out_off, 0, h, 0, s0.cuda_stream)
        p2.eval_device(d_in.data_ptr(), in_off, out.data_ptr(), out_off, h, B, 0, s1.cuda_stream)

    for mode, out in zip(("whole", "halves_same_code", "halves_two_codes"), outs):
        times = []
        for it in range(args.steps + 3):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s0)
            s1.wait_event(e0)
            run(mode, out)
            j = torch.cuda.Event()
            j.record(s1)
            s0.wait_event(j)
            e1.record(s0)
            torch.cuda.synchronize()
            if it >= 3:
                times.append(e0.elapsed_time(e1))
        print(json.dumps({"probe": "codecopy", "mode": mode, "batch": B, "alt": args.alt,
                          "ms_median": float(np.median(times)), "ms_min": float(np.min(times))}), flush=True)
    ref = outs[0].cpu().numpy()
    for mode, out in zip(("halves_same_code", "halves_two_codes"), outs[1:]):
        same = bool(np.array_equal(ref.view(np.uint64), out.cpu().numpy().view(np.uint64)))
        print(json.dumps({"probe": "codecopy", "mode": mode, "bitwise_equal_to_whole": same}), flush=True)


if __name__ == "__main__":
    main()
