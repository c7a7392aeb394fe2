#!/bin/bash
# humanoid_rbd (config 2) at scale: 2-3 team CTAs per SM (smaller teams, half the smem) vs 1
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 10 --workload humanoid_rbd --batch 4096 65536"
$S > $O/sweep49.jsonl 2>$O/sweep49.err
for spec in "team=8 min_blocks=2 team_smem=100000" "team=6 min_blocks=2 team_smem=100000" "team=12 min_blocks=2 team_smem=100000" "team=4 min_blocks=3 team_smem=65000" "team=8"; do
  $S --check 8 --grid $spec >> $O/sweep49.jsonl 2>>$O/sweep49.err
done
echo done
