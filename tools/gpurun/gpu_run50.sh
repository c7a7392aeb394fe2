#!/bin/bash
# team width vs batch regime (one wave vs many) for the team-mode tapes
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 10"
for w in srbm_mpc ldlt_57 quad_step humanoid_rbd; do
  $S --workload $w --batch 512 4096 32768 --grid team=8,12,16 >> $O/sweep50.jsonl 2>>$O/sweep50.err
done
echo done
