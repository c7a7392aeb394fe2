#!/bin/bash
# new reference-mirroring parity tests + batch-size scan (metric: batch 1e2..1e6)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "serial_bitwise or shuffling or nan_and_inf" > $O/pytest30.log 2>&1; echo "rc=$?" >> $O/pytest30.log
S="timeout 900 python tools/sweep.py --steps 5 --warmup 2"
$S --workload srbm_mpc --batch 100 1000 4096 10000 65536 100000 > $O/scan30.jsonl 2>$O/scan30.err
$S --workload humanoid_rbd --batch 100 1000 4096 10000 65536 100000 1000000 >> $O/scan30.jsonl 2>>$O/scan30.err
$S --workload cartpole_rk4 pendulum --batch 100 1000 4096 10000 100000 1000000 >> $O/scan30.jsonl 2>>$O/scan30.err
$S --workload srbm_mpc --batch 1000000 --steps 2 --warmup 1 >> $O/scan30.jsonl 2>>$O/scan30.err
echo done
