#!/bin/bash
# small batches: spread a few instances over many CTAs so that the SMs of a GPC share
# instruction-cache (L1.5) fills (VSB_IPC_FILL=1 + VSB_IPC_MIN floor)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 100 500 1000 2000"
$S | sed 's/^{/{"fill": 0, /' > $O/sweep45.jsonl 2>$O/sweep45.err
for mn in 1 4 8; do VSB_IPC_FILL=1 VSB_IPC_MIN=$mn $S --check 8 | sed "s/^{/{\"fill\": 1, \"ipc_min\": $mn, /" >> $O/sweep45.jsonl 2>>$O/sweep45.err; done
echo done
