#!/bin/bash
# roa_scan wall time after memoising the invariant split (no graph capture for one-shot calls)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_quadsim.py -m gpu -q > $O/pytest71.log 2>&1; echo "rc=$?" >> $O/pytest71.log
timeout 600 python - >> $O/roa71.jsonl 2>>$O/roa71.err <<'PY'
import json, time, numpy as np, torch, workloads
from paper_2408_09662_b200 import quadsim as qs
tape = workloads.load_tape("quad_step")
mx = np.linspace(-2, 2, 100); mw = np.linspace(-0.1, 0.1, 100); um = np.linspace(2, 10, 10)
qs.roa_scan(mx[:2], mw[:2], um[:2], steps=500, tape=tape)   # compile / warm-up
for rep in range(3):
    t0 = time.perf_counter(); masks = qs.roa_scan(mx, mw, um, steps=500, tape=tape); t1 = time.perf_counter()
    print(json.dumps({"what": "roa_scan 100x100 grid x 10 thrust limits (1e5 rollouts) x 500 steps, wall incl. setup + D2H",
                      "s": t1 - t0, "env_steps_per_s": 1e5 * 500 / (t1 - t0), "stable_frac": float(np.mean(masks))}))
PY
echo done
