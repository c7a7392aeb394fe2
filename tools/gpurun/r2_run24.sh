#!/bin/bash
# round 2, run 24: chunk size and team width under the remat-128 default (spills now fall
# to 0.2-0.5 KB/thread at <= 18k ops per chunk), srbm_mpc B=4096, parity on 16 rows
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 30 --check 16 --workload srbm_mpc"
{
  for rep in 1 2; do
    $S --batch 4096
    $S --batch 4096 --grid chunk_ops=12000,15000,18000,21000,30000,36000
    $S --batch 4096 --grid team=12
    $S --batch 4096 --grid team=12 chunk_ops=18000,30000,40000
  done
} > $O/r2_24_sweep.jsonl 2> $O/r2_24_sweep.err

# the large-batch shape (8-warp teams x 2 groups, remat 256) with smaller chunks: spills
# 24.9 KB/thread at the default 24k ops, 2.2 KB at 12k
{
  for rep in 1 2; do
    VSB_REMAT_GAP=256 $S --batch 65536 --grid team=8 groups=2
    VSB_REMAT_GAP=256 $S --batch 65536 --grid team=8 groups=2 chunk_ops=12000,15000,18000
  done
} > $O/r2_24_wide.jsonl 2> $O/r2_24_wide.err
