#!/bin/bash
# fused closed-loop rollout kernel (state in registers, one launch): parity + throughput
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rollout" > $O/pytest60.log 2>&1; echo "rc=$?" >> $O/pytest60.log
for w in "quad_step 10000" "quad_step 1000000" "pendulum 1000000" "cartpole_rk4 1000000"; do
  set -- $w
  timeout 600 python tools/rollout_bench.py --workload $1 --batch $2 --steps 100 >> $O/rollout60.jsonl 2>>$O/rollout60.err
done

timeout 600 python tools/rollout_bench.py --workload pendulum --batch 1000000 --steps 100 --fused off >> $O/rollout60.jsonl 2>>$O/rollout60.err
timeout 600 python tools/rollout_bench.py --workload quad_step --batch 10000 --steps 100 --fused off >> $O/rollout60.jsonl 2>>$O/rollout60.err
echo done
