#!/bin/bash
# team x groups x cluster sweep (instruction-fetch sharing / cross-SM teams), srbm_mpc
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc"
for spec in "team=16" "team=16 groups=4 cluster=4" "team=8 groups=2 cluster=2" "team=16 cluster=2" "team=16 phase_cost=32" \
            "team=16 groups=2 cluster=2 phase_cost=32" "team=16 groups=8 cluster=8" "team=16 groups=2 cluster=2" "team=8 groups=4 cluster=2"; do
  $S --batch 4096 --check 16 --grid $spec >> $O/sweep10.jsonl 2>>$O/sweep10.err
done
for spec in "team=16" "team=8 groups=2" "team=4 groups=4" "team=8 groups=4 cluster=2" "team=16 groups=4 cluster=4"; do
  $S --batch 65536 --grid $spec >> $O/sweep10.jsonl 2>>$O/sweep10.err
done
echo done
