#!/bin/bash
# TMA tile pipeline vs classic kernel across batch sizes (when does the persistent pipeline pay?)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/sweep.py --steps 10 --workload cartpole_rk4 pendulum --batch 1000 4096 10000 30000 100000 300000 1000000 --grid bulk_io=0,-1 > $O/sweep32.jsonl 2>$O/sweep32.err
echo done
