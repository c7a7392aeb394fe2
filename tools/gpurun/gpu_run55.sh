#!/bin/bash
# device-resident rollouts (§8 f1) with the current generator
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python tools/rollout_bench.py --batch 10000 --steps 100 > $O/rollout55.jsonl 2> $O/rollout55.err
timeout 600 python tools/rollout_bench.py --workload pendulum --batch 1000000 --steps 100 >> $O/rollout55.jsonl 2>> $O/rollout55.err
timeout 600 python tools/rollout_bench.py --workload cartpole_rk4 --batch 1000000 --steps 100 >> $O/rollout55.jsonl 2>> $O/rollout55.err
echo done
