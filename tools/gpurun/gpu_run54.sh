#!/bin/bash
# scheduler cost model: charge cross-warp operand loads to the consuming warp (VSB_XCOST)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for x in 0 0.5 1; do
  if [ $x = 0 ]; then unset VSB_XCOST; else export VSB_XCOST=$x; fi
  timeout 600 python tools/sweep.py --steps 20 --workload srbm_mpc --batch 512 4096 --grid team=16 | sed "s/^{/{\"xcost\": $x, /" >> $O/sweep54.jsonl 2>>$O/sweep54.err
  timeout 600 python tools/sweep.py --steps 20 --workload ldlt_57 humanoid_rbd --batch 4096 --grid team=12 | sed "s/^{/{\"xcost\": $x, /" >> $O/sweep54.jsonl 2>>$O/sweep54.err
done
echo done
