#!/bin/bash
# mid-size thread-mode tape (ldlt_12, 1.35k ops): CTAs per SM
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/sweep.py --steps 10 --workload ldlt_12 --batch 65536 1000000 --check 8 --grid min_blocks=1,2,3,4,6,8 > $O/sweep57.jsonl 2>$O/sweep57.err
echo done
