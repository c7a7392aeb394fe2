#!/bin/bash
# trajectory-free rollouts (roa_scan mode): parity + 1e6-env throughput
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rollout" > $O/pytest62.log 2>&1; echo "rc=$?" >> $O/pytest62.log
timeout 600 python tools/rollout_bench.py --workload quad_step --batch 1000000 --steps 100 --shared-theta --no-record >> $O/rollout62.jsonl 2>>$O/rollout62.err
timeout 600 python tools/rollout_bench.py --workload quad_step --batch 10000 --steps 100 --shared-theta --no-record >> $O/rollout62.jsonl 2>>$O/rollout62.err
timeout 600 python tools/rollout_bench.py --workload pendulum --batch 1000000 --steps 100 --no-record >> $O/rollout62.jsonl 2>>$O/rollout62.err
timeout 600 python tools/rollout_bench.py --workload cartpole_rk4 --batch 1000000 --steps 100 --no-record >> $O/rollout62.jsonl 2>>$O/rollout62.err
echo done
