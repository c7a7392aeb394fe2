#!/bin/bash
# defaults after r19 (thread-mode occupancy, trig fast path in thread mode only), warm-link e2e
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for pb in 4194304 2097152 8388608; do
  VSB_HOST_PIECE_BYTES=$pb timeout 300 python tools/e2e_probe.py >> $O/e2e22.jsonl 2>>$O/e2e22.err
done
timeout 900 python bench.py > $O/bench22.json 2> $O/bench22.err
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest22.log 2>&1; echo "pytest rc=$?" >> $O/pytest22.log
echo done
