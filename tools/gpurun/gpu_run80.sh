#!/bin/bash
# rollout kernel: 16-byte vector stores of each recorded step -- parity + throughput
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_quadsim.py -m gpu -q -x -k "rollout or roa or quadsim or sweep" > $O/pytest80.log 2>&1; echo "rc=$?" >> $O/pytest80.log
for w in "quad_step 1000000 --shared-theta" "quad_step 10000 --shared-theta" "quad_step 1000000 --shared-theta --no-record" "pendulum 1000000" "cartpole_rk4 1000000"; do
  set -- $w
  timeout 600 python tools/rollout_bench.py --workload $1 --batch $2 --steps 100 $3 $4 >> $O/rollout80.jsonl 2>>$O/rollout80.err
done
echo done
