#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 300 python tools/trig_bench.py > $O/trig39.json 2> $O/trig39.err
timeout 900 python tools/sweep.py --steps 10 --workload cartpole_rk4 pendulum --batch 1000000 --check 64 > $O/sweep39.jsonl 2>$O/sweep39.err
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest39.log 2>&1; echo "pytest rc=$?" >> $O/pytest39.log
echo done
