#!/bin/bash
# first GPU session: environment, parity tests, smoke, bench lines
cd "$GRAFT_REPO_ROOT"
O=gpurun_out
mkdir -p $O
{ nproc; lscpu | grep -E 'Model name|Socket|Core|Thread|NUMA node\(s\)'; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; free -g | head -2; } > $O/env.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-w1 > $O/bench_srbm.json 2> $O/bench_srbm.err
timeout 300 python bench.py --workload cartpole_rk4 --batch 1000000 --steps 20 --cpu-seconds 5 > $O/bench_cartpole.json 2> $O/bench_cartpole.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
echo done
