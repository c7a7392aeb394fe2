#!/bin/bash
# trig share of the small-tape HBM kernels: SIN/COS rewritten to NEG (timing only)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/op_probe.py --workload pendulum --batch 1000000 4000000 --swap SIN=NEG COS=NEG > $O/probe68.jsonl 2>$O/probe68.err
timeout 900 python tools/op_probe.py --workload cartpole_rk4 --batch 1000000 --swap SIN=NEG COS=NEG DIV=MUL >> $O/probe68.jsonl 2>>$O/probe68.err
echo done
