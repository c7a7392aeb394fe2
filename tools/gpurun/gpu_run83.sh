#!/bin/bash
# ldlt_12 (latency-bound thread kernel at 6 % occupancy): team widths 2/4/8 vs thread mode
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1200 python tools/sweep.py --steps 10 --workload ldlt_12 --batch 65536 1000000 --check 8 --grid team=1,2,4,8 > $O/sweep83.jsonl 2>$O/sweep83.err
echo done
