#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/ifetch_bench.py --ops 8000 > $O/ifetch.jsonl 2> $O/ifetch.err
S="timeout 900 python tools/sweep.py --steps 10"
$S --workload srbm_mpc --batch 4096 --grid team=4,12 > $O/sweep4_srbm.jsonl 2>&1
$S --workload srbm_mpc --batch 4096 --grid team=8 chunk_ops=8000 >> $O/sweep4_srbm.jsonl 2>&1
echo done
