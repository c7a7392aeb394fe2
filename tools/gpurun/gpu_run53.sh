#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "soa or fp32" > $O/pytest53.log 2>&1; echo "rc=$?" >> $O/pytest53.log
echo done
