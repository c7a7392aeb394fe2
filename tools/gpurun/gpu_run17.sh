#!/bin/bash
# batch-size scan of the team kernel (fetch vs critical path), bench line with secondary points,
# ncu of the thread-mode cartpole kernel at 1e6
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 512 1024 2048 4096 8192 --grid team=16 > $O/sweep17.jsonl 2>$O/sweep17.err
timeout 900 python bench.py > $O/bench17.json 2> $O/bench17.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vsk_ -c 1 -o $O/prof17_cartpole \
  python tools/sweep.py --workload cartpole_rk4 --batch 1000000 --steps 1 --warmup 0 > $O/ncu17.log 2>&1
echo done
