#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
VSB_TRACE=1 timeout 300 python tools/e2e_probe.py --calls 5 > $O/e2e26.out 2> $O/e2e26.err
timeout 300 python tools/e2e_probe.py --workload cartpole_rk4 --batch 1000000 >> $O/e2e26.out 2>> $O/e2e26.err
timeout 900 python bench.py > $O/bench26.json 2> $O/bench26.err
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest26.log 2>&1; echo "pytest rc=$?" >> $O/pytest26.log
echo done
