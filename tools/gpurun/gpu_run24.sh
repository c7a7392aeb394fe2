#!/bin/bash
# persistent host-path workspace (no per-call pool allocations across streams)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for pb in 16777216 4194304 2097152 1048576; do
  VSB_HOST_PIECE_BYTES=$pb timeout 300 python tools/e2e_probe.py >> $O/e2e24.jsonl 2>>$O/e2e24.err
done
VSB_HOST_PIECE_BYTES=4194304 timeout 300 python tools/e2e_probe.py --workload cartpole_rk4 --batch 1000000 >> $O/e2e24.jsonl 2>>$O/e2e24.err
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest24.log 2>&1; echo "pytest rc=$?" >> $O/pytest24.log
echo done
