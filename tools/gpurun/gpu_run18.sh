#!/bin/bash
# table-based correctly rounded sin/cos fast path: parity suite + small-tape throughput + bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest18.log 2>&1; echo "pytest rc=$?" >> $O/pytest18.log
timeout 600 python tools/sweep.py --steps 10 --workload cartpole_rk4 pendulum --batch 1000000 --check 64 > $O/sweep18.jsonl 2>$O/sweep18.err
timeout 600 python tools/sweep.py --steps 10 --workload humanoid_rbd --batch 65536 --check 64 >> $O/sweep18.jsonl 2>>$O/sweep18.err
timeout 900 python bench.py > $O/bench18.json 2> $O/bench18.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vsk_ -c 1 -o $O/prof18_cartpole \
  python tools/sweep.py --workload cartpole_rk4 --batch 1000000 --steps 1 --warmup 0 > $O/ncu18.log 2>&1
echo done
