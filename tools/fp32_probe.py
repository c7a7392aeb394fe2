#!/usr/bin/env python
"""fp32-mode error distribution per workload (GPU box): |g32 - r64| / max(|r64|, 1)
against the fp64 CPU oracle on seeded inputs; one JSON line per workload with the
max, 99.9th percentile and median error (the numbers the per-config fp32
tolerances in tests/test_gpu_contract.py are stated from)."""

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

B = {"pendulum": 4096, "cartpole_rk4": 4096, "ldlt_12": 2048, "ldlt_25": 1024, "ldlt_57": 256, "quad_step": 1024,
     "unicycle_mpc": 512, "srbm_mpc": 512, "rbd_chain12": 256, "humanoid_rbd": 2048}
for name, b in B.items():
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, b, seed=77)
    ref = oracle.batch_eval(tape, ins, n_threads=8)
    f = Function(tape, dtype=torch.float32)
    outs = f(*[torch.tensor(v, dtype=torch.float32, device="cuda") for v in ins])
    errs = []
    for o, r in zip(outs, ref):
        g = o.double().cpu().numpy()
        with np.errstate(invalid="ignore", over="ignore"):
            errs.append((np.abs(g - r) / np.maximum(np.abs(r), 1.0)).ravel())
    e = np.concatenate(errs)
    nonfinite = int(np.count_nonzero(~np.isfinite(e)))
    e = e[np.isfinite(e)]
    print(json.dumps({"workload": name, "batch": b, "max": float(e.max()), "p999": float(np.quantile(e, 0.999)),
                      "median": float(np.median(e)), "nonfinite": nonfinite}), flush=True)
