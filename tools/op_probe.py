"""Upper bound of an opcode's share of a kernel step: time a workload as-is and
with every row of one opcode rewritten to a cheap opcode (results are wrong;
timing only).

    python tools/op_probe.py --workload srbm_mpc --batch 4096 --swap DIV=MUL
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="srbm_mpc")
    ap.add_argument("--batch", type=int, nargs="+", default=[4096])
    ap.add_argument("--swap", nargs="+", default=["DIV=MUL"])
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()

    import paper_2408_09662_b200 as vsb
    import workloads
    from paper_2408_09662_b200.tape import InstructionTape, OpCode
    from sweep import time_plan

    tape = workloads.load_tape(args.workload)
    variants = [("as_is", tape)]
    for sw in args.swap:
        a, b = sw.split("=")
        code, values = tape.packed()
        code = code.copy()
        code[code[:, 0] == int(OpCode[a]), 0] = int(OpCode[b])
        variants.append((sw, InstructionTape(tape.name, code, values, tape.n_w, tape.input_sparsity,
                                             tape.output_sparsity)))
    for B in args.batch:
        inputs = workloads.make_inputs(args.workload, B, seed=0)
        for name, t in variants:
            plan = vsb.Plan(t)
            ms, _ = time_plan(plan, t, inputs, B, args.steps, 3)
            print(json.dumps({"workload": args.workload, "batch": B, "variant": name, "ms": ms,
                              "code_bytes": plan.info["code_bytes"]}), flush=True)


if __name__ == "__main__":
    main()
