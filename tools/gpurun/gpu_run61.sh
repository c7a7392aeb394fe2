#!/bin/bash
# rollouts: pre tape once per distinct parameter row (dedup) -- parity + quad_step with a broadcast theta
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rollout" > $O/pytest61.log 2>&1; echo "rc=$?" >> $O/pytest61.log
for b in 10000 1000000; do
  timeout 600 python tools/rollout_bench.py --workload quad_step --batch $b --steps 100 --shared-theta >> $O/rollout61.jsonl 2>>$O/rollout61.err
  timeout 600 python tools/rollout_bench.py --workload quad_step --batch $b --steps 100 --shared-theta --dedup off >> $O/rollout61.jsonl 2>>$O/rollout61.err
done
echo done
