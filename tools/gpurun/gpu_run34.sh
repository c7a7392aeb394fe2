#!/bin/bash
# config 5 (large-tape stress) with the current generator: fp64 + fp32, error distribution
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 5 --warmup 2 --check 64"
$S --workload rbd_chain12 ldlt_57 --batch 4096 > $O/sweep34.jsonl 2>$O/sweep34.err
$S --workload rbd_chain12 ldlt_57 srbm_mpc humanoid_rbd --batch 4096 --dtype float32 >> $O/sweep34.jsonl 2>>$O/sweep34.err
$S --workload rbd_chain12 --batch 4096 --grid team=8,32 >> $O/sweep34.jsonl 2>>$O/sweep34.err
echo done
