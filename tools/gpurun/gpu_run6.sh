#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu6.log 2>&1
S="timeout 900 python tools/sweep.py --steps 10"
$S --workload srbm_mpc --batch 4096 --grid team=8,12,16 > $O/sweep6.jsonl 2>&1
$S --workload cartpole_rk4 --batch 1000000 --grid min_blocks=1,8 >> $O/sweep6.jsonl 2>&1
$S --workload cartpole_rk4 --batch 1000000 --grid min_blocks=8 libdevice_trig=1 >> $O/sweep6.jsonl 2>&1
$S --workload cartpole_rk4 --batch 1000000 --grid team=4 >> $O/sweep6.jsonl 2>&1
$S --workload quad_step --batch 4096 --grid team=1,8,16 >> $O/sweep6.jsonl 2>&1
$S --workload humanoid_rbd --batch 4096 65536 --grid team=1,8 >> $O/sweep6.jsonl 2>&1
$S --workload ldlt_25 unicycle_mpc --batch 4096 >> $O/sweep6.jsonl 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-w1 > $O/bench6.json 2> $O/bench6.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches6.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu6_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vsk_ -s 8 -c 1 -o $O/prof6_srbm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu6_full.log 2>&1
echo done
