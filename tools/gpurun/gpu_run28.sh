#!/bin/bash
# persistent TMA tile pipeline (thread mode): correctness + throughput
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tma" > $O/pytest28_tma.log 2>&1; echo "rc=$?" >> $O/pytest28_tma.log
timeout 900 python tools/sweep.py --steps 10 --workload pendulum cartpole_rk4 --batch 1000000 --check 64 --grid bulk_io=0,-1 min_blocks=8,12,16 > $O/sweep28.jsonl 2>$O/sweep28.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:_tma -c 1 -o $O/prof28_pendulum_tma \
  python tools/sweep.py --workload pendulum --batch 1000000 --steps 1 --warmup 0 > $O/ncu28.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest28.log 2>&1; echo "pytest rc=$?" >> $O/pytest28.log
echo done
