#!/usr/bin/env python
"""First op where the GPU and the oracle disagree (GPU box; diagnostic).

    python tools/tape_bisect.py --fuzz acc 57 4096 --rows 665

Instruments the tape so that every arithmetic row's result is also an output (one extra
output array, one nonzero per arithmetic row), evaluates it on the GPU and with the oracle
on the same inputs, and prints for each requested row the first arithmetic row whose value
differs (NaN == NaN), with its opcode and operand values on both sides.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))

NAMES = ("CONST INPUT OUTPUT ASSIGN ADD SUB MUL DIV NEG EXP LOG POW SQRT SQ SIN COS TAN ATAN2 FABS FMIN FMAX "
         "STEP IF_ELSE").split()
AR = [0, 0, 1, 1, 2, 2, 2, 2, 1, 1, 1, 2, 1, 1, 1, 1, 1, 2, 1, 2, 2, 1, 3]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fuzz", nargs=3, metavar=("FAM", "IDX", "B"))
    ap.add_argument("--workload", nargs=2, metavar=("NAME", "B"))
    ap.add_argument("--rows", type=int, nargs="+", required=True)
    ap.add_argument("--opts", default="{}")
    args = ap.parse_args()
    import oracle
    from paper_2408_09662_b200 import BatchWorkspace, InstructionTape, batch_eval

    if args.fuzz:
        from test_acceptance_fuzz import _golden, _tapes, inputs_for

        fam, idx, B = args.fuzz[0], int(args.fuzz[1]), int(args.fuzz[2])
        tape = _tapes(_golden(), fam)[idx]
        ins = inputs_for(fam, idx, tape.nnz_in, B)
    else:
        import workloads

        tape = workloads.load_tape(args.workload[0])
        B = int(args.workload[1])
        ins = workloads.make_inputs(args.workload[0], B, seed=5)
    ins = [v[args.rows] for v in ins]   # only the rows of interest (row order kept)
    code, vals = tape.packed()
    arith = [r for r in range(code.shape[0]) if code[r, 0] > 3]
    extra = len(tape.nnz_out)
    rows = []
    for r in range(code.shape[0]):
        rows.append(code[r].tolist())
        if code[r, 0] > 3:   # trace the result of this arithmetic row
            rows.append([2, extra, int(code[r, 1]), arith.index(r), -1])
    t2 = InstructionTape(tape.name + "_traced", np.array(rows, dtype=np.int32),
                         np.array([vals[r] for r in range(code.shape[0]) for _ in range(2 if code[r, 0] > 3 else 1)]),
                         tape.n_w, list(tape.nnz_in), list(tape.nnz_out) + [len(arith)])
    ws = BatchWorkspace(t2, len(args.rows))
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    batch_eval(t2, ws, plan_options=json.loads(args.opts) or None)
    got = ws.output_matrix(extra)
    ref = oracle.batch_eval(t2, ins)[extra]
    for k, row in enumerate(args.rows):
        g, r = got[k], ref[k]
        same = (g == r) | (np.isnan(g) & np.isnan(r))
        bad = np.where(~same)[0]
        if bad.size == 0:
            print(json.dumps({"row": row, "first_diff": None}))
            continue
        a = bad[0]
        rr = arith[a]
        op = int(code[rr, 0])
        operands = []
        for s in code[rr, 2:2 + AR[op]]:
            # value of the operand slot: the last traced row writing that slot before rr
            prev = [x for x in arith[:a] if code[x, 1] == s]
            operands.append({"slot": int(s), "gpu": float(got[k][arith.index(prev[-1])]) if prev else None,
                             "ref": float(ref[k][arith.index(prev[-1])]) if prev else None})
        print(json.dumps({"row": row, "first_diff_row": int(rr), "op": NAMES[op], "gpu": float(g[a]), "ref": float(r[a]),
                          "operands": operands, "n_diff": int(bad.size)}))


if __name__ == "__main__":
    main()
