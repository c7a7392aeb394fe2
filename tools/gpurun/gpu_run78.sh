#!/bin/bash
# ncu --set full of the fused closed-loop rollout kernel (quad_step step tape, 1e6 envs x 100 steps, recorded)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:_roll -c 1 -o $O/roll78 -f \
  python tools/rollout_bench.py --workload quad_step --batch 1000000 --steps 100 --shared-theta > $O/ncu78.log 2>&1
ncu -i $O/roll78.ncu-rep --page raw --csv > $O/roll78_raw.csv 2>/dev/null
ncu -i $O/roll78.ncu-rep --page details --csv > $O/roll78_details.csv 2>/dev/null
echo done
