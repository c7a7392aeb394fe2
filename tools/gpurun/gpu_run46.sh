#!/bin/bash
# tiny-batch spread default + full GPU suite + small-batch scan
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/sweep.py --steps 10 --workload srbm_mpc humanoid_rbd --batch 1 32 100 300 500 --check 8 > $O/sweep46.jsonl 2>$O/sweep46.err
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest46.log 2>&1; echo "pytest rc=$?" >> $O/pytest46.log
echo done
