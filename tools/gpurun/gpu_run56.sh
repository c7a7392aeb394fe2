#!/bin/bash
# full workload matrix with the final defaults: every workload x B in {1e3, 4096, 65536}, fp64 and fp32, oracle check
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 1200 python tools/sweep.py --steps 5 --warmup 2 --check 16"
$S --workload example pendulum cartpole_rk4 ldlt_12 ldlt_25 ldlt_57 quad_step unicycle_mpc srbm_mpc rbd_chain12 humanoid_rbd --batch 1000 4096 65536 > $O/matrix56.jsonl 2>$O/matrix56.err
$S --dtype float32 --workload cartpole_rk4 ldlt_57 quad_step srbm_mpc rbd_chain12 humanoid_rbd --batch 4096 65536 >> $O/matrix56.jsonl 2>>$O/matrix56.err
echo done
