#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests/test_acceptance_fuzz.py -m gpu -q -rf -k "gpu and acc" > $O/r2_17b_acc.log 2>&1; echo "acc rc=$?"
tail -5 $O/r2_17b_acc.log
bash tools/gpurun/r2_run18.sh; echo "sweep done"
