#!/bin/bash
# round 2, run 21: rematerialised reloads (VSB_REMAT_GAP) for the one-wave 16-warp shape of
# srbm_mpc (B=4096; spills 6.5 -> 5.4 KB/thread at compile time), parity on 16 rows
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 30 --check 16 --workload srbm_mpc --batch 4096"
{
  for rep in 1 2; do
    $S
    for g in 64 128 256 512; do VSB_REMAT_GAP=$g $S | sed "s/^{/{\"remat\": $g, /"; done
  done
} > $O/r2_21_sweep.jsonl 2> $O/r2_21_sweep.err
