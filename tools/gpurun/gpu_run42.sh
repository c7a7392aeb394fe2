#!/bin/bash
# large-batch srbm in thread mode: smaller chunks x more CTAs/SM vs team 16
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 5 --warmup 2 --workload srbm_mpc --batch 65536"
$S --grid team=16 > $O/sweep42.jsonl 2>$O/sweep42.err
for spec in "team=1 chunk_ops=3000 min_blocks=4" "team=1 chunk_ops=3000 min_blocks=8" "team=1 chunk_ops=6000 min_blocks=4" "team=1 chunk_ops=1500 min_blocks=6" "team=1"; do
  $S --check 8 --grid $spec >> $O/sweep42.jsonl 2>>$O/sweep42.err
done
echo done
