#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
python tools/dump_random.py > $O/dump_random.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu2.log 2>&1
timeout 900 python tools/sweep.py --workload srbm_mpc --batch 4096 --grid block=32,64,128 chunk_ops=2000,4000,8000 > $O/sweep_srbm.jsonl 2>&1
timeout 600 python tools/sweep.py --workload cartpole_rk4 --batch 1000000 --grid block=128,256 min_blocks=1,4,8 > $O/sweep_cart.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_srbm.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vsk_ -s 30 -c 1 -o $O/prof_srbm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_srbm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vsk_ -s 3 -c 1 -o $O/prof_cart python bench.py --workload cartpole_rk4 --batch 1000000 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_cart.log 2>&1
echo done
