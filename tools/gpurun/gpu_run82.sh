#!/bin/bash
# ncu --set full of the thread-mode TMA tile kernel: ldlt_12 (block 64) and cartpole_rk4 at B=1e6
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for w in ldlt_12 cartpole_rk4; do
timeout 900 ncu --set full --clock-control none -k regex:_tma -c 1 -o $O/tma82_$w -f \
  python tools/sweep.py --steps 1 --warmup 1 --workload $w --batch 1000000 > $O/ncu82_$w.log 2>&1
ncu -i $O/tma82_$w.ncu-rep --page details --csv > $O/tma82_${w}_details.csv 2>/dev/null
ncu -i $O/tma82_$w.ncu-rep --page raw --csv > $O/tma82_${w}_raw.csv 2>/dev/null
done
echo done
