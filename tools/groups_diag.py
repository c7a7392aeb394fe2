#!/usr/bin/env python
"""Which rows / outputs of a grouped team plan disagree with the oracle (GPU box, diagnostic).

    python tools/groups_diag.py ldlt_57 4096 '{"team": 8, "groups": 2}'
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))

import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2408_09662_b200 import Function  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
opts = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
tape = workloads.load_tape(name)
ins = workloads.make_inputs(name, B, seed=5)
f = Function(tape, **opts)
runs = []
for rep in range(3):
    outs = f(*[torch.tensor(v, device="cuda") for v in ins])
    torch.cuda.synchronize()
    runs.append([o.cpu().numpy() for o in outs])
ref = oracle.batch_eval(tape, ins, n_threads=8)
for j, r in enumerate(ref):
    g = runs[0][j]
    with np.errstate(invalid="ignore"):
        e = np.abs(g - r) / np.maximum(np.abs(r), 1.0)
    bad = e > 1e-12
    rows = np.where(bad.any(axis=1))[0]
    cols = np.where(bad.any(axis=0))[0]
    same = all(np.array_equal(runs[0][j], runs[k][j], equal_nan=True) for k in (1, 2))
    print(json.dumps({"out": j, "bad_elems": int(bad.sum()), "of": int(bad.size), "bad_rows": int(rows.size),
                      "bad_cols": cols[:40].tolist(), "n_bad_cols": int(cols.size),
                      "rows_head": rows[:20].tolist(), "lane_hist": np.bincount(rows % 64, minlength=64).tolist(),
                      "deterministic_over_3_runs": same, "max_err": float(np.nanmax(e))}))
