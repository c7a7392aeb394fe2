#!/bin/bash
# shared-reciprocal division (DIVR) in thread-mode kernels: bitwise tests + A/B timing
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_divr.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest65.log 2>&1; echo "rc=$?" >> $O/pytest65.log
for r in 1 0; do
  VSB_DIV_RECIP=$r VSB_CACHE_DIR=/tmp/vsbc$r timeout 900 python tools/sweep.py --steps 20 --workload ldlt_12 cartpole_rk4 --batch 65536 1000000 --check 8 --grid block=128 > $O/sweep65_r$r.jsonl 2>$O/sweep65_r$r.err
done
echo done
