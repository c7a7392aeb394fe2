#!/bin/bash
# persisting-L2 window on the chunk scratch (experiment)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 4096 65536"
$S | sed 's/^{/{"l2p": 0, /' > $O/sweep36.jsonl 2>$O/sweep36.err
for mb in 32 64 96; do VSB_L2_PERSIST=$mb $S | sed "s/^{/{\"l2p\": $mb, /" >> $O/sweep36.jsonl 2>>$O/sweep36.err; done
echo done
