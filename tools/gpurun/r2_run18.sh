#!/bin/bash
# round 2, run 18: chunk size and phase capacity under the local-search schedule
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 1200 python tools/sweep.py --steps 20 --check 8"
{
  $S --workload srbm_mpc --batch 4096 --grid chunk_ops=18000,30000,36000
  $S --workload srbm_mpc --batch 4096
  $S --workload srbm_mpc --batch 4096 --grid phase_cost=64,80
  $S --workload humanoid_rbd --batch 4096 65536 --grid phase_cost=48,64,96,128
} > $O/r2_18_sweep.jsonl 2> $O/r2_18_sweep.err
