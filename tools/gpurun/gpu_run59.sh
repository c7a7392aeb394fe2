#!/bin/bash
# loop-invariant hoisting in device rollouts: parity (hoisted == unhoisted bitwise, vs host loop) + throughput
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "rollout" > $O/pytest59.log 2>&1; echo "rc=$?" >> $O/pytest59.log
for h in on off; do
  timeout 600 python tools/rollout_bench.py --workload quad_step --batch 10000 --steps 100 --hoist $h >> $O/rollout59.jsonl 2>>$O/rollout59.err
done
timeout 600 python tools/rollout_bench.py --workload quad_step --batch 100000 --steps 100 --hoist on >> $O/rollout59.jsonl 2>>$O/rollout59.err
timeout 600 python tools/rollout_bench.py --workload quad_step --batch 1000000 --steps 100 --hoist on >> $O/rollout59.jsonl 2>>$O/rollout59.err
echo done
