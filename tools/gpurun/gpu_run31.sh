#!/bin/bash
# per-chunk kernel times vs phase length (team 16, srbm B=4096)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for pc in 32 48 64 96 128; do
  timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 4096 --grid team=16 phase_cost=$pc >> $O/sweep31.jsonl 2>>$O/sweep31.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vsk_ --csv --log-file $O/launch31_pc$pc.csv \
    python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 2 --warmup 1 --grid team=16 phase_cost=$pc > /dev/null 2>&1
done
echo done
