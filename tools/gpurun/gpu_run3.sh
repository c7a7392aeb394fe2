#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu3.log 2>&1
S="timeout 900 python tools/sweep.py --steps 10"
$S --workload srbm_mpc --batch 4096 --grid team=8,16 > $O/sweep3_srbm.jsonl 2>&1
$S --workload srbm_mpc --batch 4096 --grid team=8 phase_cost=128 >> $O/sweep3_srbm.jsonl 2>&1
$S --workload srbm_mpc --batch 4096 --grid team=16 phase_cost=64 >> $O/sweep3_srbm.jsonl 2>&1
$S --workload humanoid_rbd --batch 4096 65536 --grid team=1,8 > $O/sweep3_other.jsonl 2>&1
$S --workload quad_step --batch 4096 --grid team=1,16 >> $O/sweep3_other.jsonl 2>&1
$S --workload ldlt_25 --batch 4096 --grid team=1,16 >> $O/sweep3_other.jsonl 2>&1
$S --workload unicycle_mpc --batch 4096 --grid team=1,8 >> $O/sweep3_other.jsonl 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench3.json 2> $O/bench3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vsk_ -s 3 -c 1 -o $O/prof3_srbm python tools/sweep.py --workload srbm_mpc --batch 4096 --grid team=8 --steps 1 --warmup 1 > $O/ncu3.log 2>&1
echo done
