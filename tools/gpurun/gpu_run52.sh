#!/bin/bash
# config 4 bench line (1e6 global batch on 1 GPU) + interleaved pairing A/B (3 x 20 steps each)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py --global-batch 1000000 --steps 5 --warmup 3 --cpu-seconds 5 --no-secondary > $O/bench52_1e6.json 2> $O/bench52_1e6.err
S="timeout 600 python tools/sweep.py --steps 20 --workload srbm_mpc --batch 4096"
for r in 1 2 3; do
  $S | sed "s/^{/{\"pair\": 0, \"rep\": $r, /" >> $O/sweep52.jsonl 2>>$O/sweep52.err
  VSB_PAIR=1 $S | sed "s/^{/{\"pair\": 1, \"rep\": $r, /" >> $O/sweep52.jsonl 2>>$O/sweep52.err
done
echo done
