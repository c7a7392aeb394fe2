#!/usr/bin/env python
"""One evaluation of a plan for compute-sanitizer (GPU box):

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py srbm_mpc 64 '{"team": 16}'
    python tools/sanitize_probe.py --fuzz acc 95 4096 '{"team": 16, "team_smem": 2048}'

Runs the plan once through the C ABI (vsb_eval_device_ptrs) on seeded inputs,
synchronises, and compares every row with the CPU oracle (exit 1 on mismatch)."""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2408_09662_b200 import Function  # noqa: E402

args = sys.argv[1:]
host = "--host" in args   # through batch_eval (the synchronous host path)
pipe = "--pipe" in args   # through BatchPipeline (3 batches, depth 2: slot reuse, overlapping copies)
args = [a for a in args if a not in ("--host", "--pipe")]
if args[0] == "--fuzz":
    from test_acceptance_fuzz import _golden, _tapes, inputs_for

    fam, idx, B = args[1], int(args[2]), int(args[3])
    tape = _tapes(_golden(), fam)[idx]
    ins = inputs_for(fam, idx, tape.nnz_in, B)
    opts = json.loads(args[4]) if len(args) > 4 else {}
else:
    import workloads

    name, B = args[0], int(args[1])
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, B, seed=5)
    opts = json.loads(args[2]) if len(args) > 2 else {}
f = Function(tape, **opts)
if pipe:
    from paper_2408_09662_b200 import BatchPipeline, BatchWorkspace

    wss = []
    for k in range(3):
        ws = BatchWorkspace(tape, B)
        for i, v in enumerate(ins):
            ws.set_input(i, v)
        wss.append(ws)
    with BatchPipeline(tape, depth=2, plan_options=opts or None) as p:
        tickets = [p.submit(ws) for ws in wss]
        for t in tickets:
            p.wait(t)
    for ws in wss[1:]:
        assert all(np.array_equal(ws.output_matrix(j), wss[0].output_matrix(j), equal_nan=True)
                   for j in range(tape.n_out))
    outs = [torch.tensor(wss[-1].output_matrix(j).copy()) for j in range(tape.n_out)]
elif host:
    from paper_2408_09662_b200 import BatchWorkspace, batch_eval

    ws = BatchWorkspace(tape, B)
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    batch_eval(tape, ws, plan_options=opts or None)
    outs = [torch.tensor(ws.output_matrix(j).copy()) for j in range(tape.n_out)]
else:
    outs = f(*[torch.tensor(v, device="cuda") for v in ins])
torch.cuda.synchronize()
ref = oracle.batch_eval(tape, ins, n_threads=8)
worst = 0.0
for o, r in zip(outs, ref):
    g = o.cpu().numpy()
    with np.errstate(invalid="ignore"):
        e = np.abs(g - r) / np.maximum(np.abs(r), 1.0)
    e[np.isnan(g) & np.isnan(r)] = 0
    worst = max(worst, float(np.nanmax(e)) if e.size else 0.0)
info = f.plan.info
print(json.dumps({"tape": tape.name, "batch": B, "opts": opts, "host": host, "pipe": pipe, "team": info["team"], "chunks": info["n_chunks"],
                  "overflow_slots": info["overflow_slots"], "max_rel_err": worst}))
sys.exit(0 if worst <= 1e-9 else 1)
