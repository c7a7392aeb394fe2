#!/bin/bash
# tiny-batch redundancy (>= 24 CTAs) + GPU suite
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/sweep.py --steps 10 --workload srbm_mpc humanoid_rbd --batch 1 8 32 100 --check 8 > $O/sweep47.jsonl 2>$O/sweep47.err
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest47.log 2>&1; echo "pytest rc=$?" >> $O/pytest47.log
echo done
