#!/bin/bash
# small-batch latency: cluster teams (team split over 2-4 SMs) vs single-CTA teams
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 100 1000"
for spec in "team=16" "team=32 cluster=2" "team=32 cluster=4" "team=16 cluster=2"; do
  $S --check 8 --grid $spec >> $O/sweep44.jsonl 2>>$O/sweep44.err
done
echo done
