#!/bin/bash
# experiment: point-to-point phase readiness (VSB_P2P=1) instead of CTA barriers in team kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
export VSB_CACHE_DIR=/tmp/vsbc_p2p
VSB_P2P=1 timeout 300 python tools/sweep.py --steps 5 --workload humanoid_rbd --batch 4096 --check 8 > $O/sweep77_smoke.jsonl 2>$O/sweep77.err
echo "smoke rc=$?" >> $O/sweep77.err
if grep -q '"ms"' $O/sweep77_smoke.jsonl; then
  VSB_P2P=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "workloads_vs_reference or team or srbm or batch_equals or shuffling or subrange" > $O/pytest77.log 2>&1; echo "rc=$?" >> $O/pytest77.log
  for z in 1 0; do
    VSB_P2P=$z timeout 900 python tools/sweep.py --steps 20 --workload srbm_mpc humanoid_rbd ldlt_57 quad_step --batch 4096 --check 8 > $O/sweep77_p$z.jsonl 2>>$O/sweep77.err
    VSB_P2P=$z timeout 900 python tools/sweep.py --steps 10 --workload humanoid_rbd srbm_mpc --batch 65536 --check 8 >> $O/sweep77_p$z.jsonl 2>>$O/sweep77.err
  done
fi
echo done
