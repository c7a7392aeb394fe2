#!/bin/bash
# round 2, run 22: rematerialised reloads across the team-mode workloads (does the srbm_mpc
# gain, 0.434 -> 0.408 ms at gap 64-128, carry over?), parity on 16 rows; code-address
# contention probe for the one-wave srbm chain
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python tools/codecopy_probe.py > $O/r2_22_codecopy.jsonl 2> $O/r2_22_codecopy.err; echo "codecopy rc=$?"
S="timeout 900 python tools/sweep.py --steps 20 --check 16"
{
  for w in "humanoid_rbd --batch 4096 65536" "rbd_chain12 --batch 4096" "ldlt_57 --batch 4096" "ldlt_25 --batch 4096" "unicycle_mpc --batch 4096"; do
    $S --workload $w
    for g in 64 128; do VSB_REMAT_GAP=$g $S --workload $w | sed "s/^{/{\"remat\": $g, /"; done
  done
} > $O/r2_22_sweep.jsonl 2> $O/r2_22_sweep.err
echo done
