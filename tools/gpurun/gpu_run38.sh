#!/bin/bash
# latency-aware op order within each warp's phase (VSB_ILP) vs program order
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10"
for ilp in 0 1; do
  if [ $ilp = 1 ]; then export VSB_ILP=1; else unset VSB_ILP; fi
  $S --workload srbm_mpc --batch 512 4096 --check 16 | sed "s/^{/{\"ilp\": $ilp, /" >> $O/sweep38.jsonl 2>>$O/sweep38.err
  $S --workload humanoid_rbd --batch 4096 65536 | sed "s/^{/{\"ilp\": $ilp, /" >> $O/sweep38.jsonl 2>>$O/sweep38.err
  $S --workload ldlt_57 --batch 4096 | sed "s/^{/{\"ilp\": $ilp, /" >> $O/sweep38.jsonl 2>>$O/sweep38.err
done
echo done
