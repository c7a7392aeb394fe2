#!/bin/bash
# 128-bit paired cross-warp exchange: A/B on srbm_mpc, parity tests
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 4096"
$S --check 16 --grid team=16 > $O/sweep15.jsonl 2>>$O/sweep15.err
VSB_NO_PAIR=1 $S --grid team=16 | sed 's/^{/{"no_pair": 1, /' >> $O/sweep15.jsonl 2>>$O/sweep15.err
$S --check 16 --grid team=12 >> $O/sweep15.jsonl 2>>$O/sweep15.err
$S --check 16 --grid team=8 >> $O/sweep15.jsonl 2>>$O/sweep15.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "team or srbm or ragged or block" > $O/pytest15.log 2>&1; echo "pytest rc=$?" >> $O/pytest15.log
echo done
