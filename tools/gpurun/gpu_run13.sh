#!/bin/bash
# round-1 measurement of the default plan: bench line, launch list, ncu --set full of the top kernel,
# dram traffic of one step, GPU tests
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py > $O/bench13.json 2> $O/bench13.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches13.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu13_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:vsk_ \
  --csv --log-file $O/traffic13.csv python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/ncu13_traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:_c2 -c 1 -o $O/prof13_default \
  python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/ncu13_full.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest13.log 2>&1; echo "pytest rc=$?" >> $O/pytest13.log
echo done
