#!/bin/bash
# chunk size around the default (24000 ops -> 5 chunks), srbm B=4096 team 16
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 4096 --grid team=16 chunk_ops=18000,21000,24000,28000,34000 > $O/sweep43.jsonl 2>$O/sweep43.err
echo done
