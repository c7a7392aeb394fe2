#!/bin/bash
# small-tape occupancy / block-size scan + ncu of pendulum at 1e6
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/sweep.py --steps 10 --workload pendulum cartpole_rk4 --batch 1000000 --grid min_blocks=8,12,16 block=64,128,256 > $O/sweep27.jsonl 2>$O/sweep27.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vsk_ -c 1 -o $O/prof27_pendulum \
  python tools/sweep.py --workload pendulum --batch 1000000 --steps 1 --warmup 0 > $O/ncu27.log 2>&1
echo done
