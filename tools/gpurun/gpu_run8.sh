#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 10"
$S --workload srbm_mpc --batch 4096 --grid team=12 chunk_ops=12000,40000,-1 > $O/sweep8.jsonl 2>&1
$S --workload srbm_mpc --batch 4096 --grid team=16 chunk_ops=-1 >> $O/sweep8.jsonl 2>&1
timeout 600 python tools/rollout_bench.py --batch 10000 --steps 100 > $O/rollout8.jsonl 2> $O/rollout8.err
timeout 600 python tools/rollout_bench.py --batch 10000 --steps 100 --team 8 >> $O/rollout8.jsonl 2>> $O/rollout8.err
timeout 600 python tools/rollout_bench.py --workload pendulum --batch 1000000 --steps 100 >> $O/rollout8.jsonl 2>> $O/rollout8.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "rollout or fp32 or known" > $O/pytest8.log 2>&1
echo done
