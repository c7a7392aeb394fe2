#!/bin/bash
# TMA kernel with in-kernel tail + size threshold; host sub-ranges; full GPU suite
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/sweep.py --steps 10 --workload cartpole_rk4 pendulum --batch 4096 100000 1000000 --grid bulk_io=0,1,-1 > $O/sweep33.jsonl 2>$O/sweep33.err
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest33.log 2>&1; echo "pytest rc=$?" >> $O/pytest33.log
echo done
