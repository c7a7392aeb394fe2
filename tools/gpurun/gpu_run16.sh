#!/bin/bash
# split (named arrive/sync) barriers vs one CTA barrier per phase; parity
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 4096"
for t in 16 12 8; do $S --check 16 --grid team=$t >> $O/sweep16.jsonl 2>>$O/sweep16.err; done
for t in 16 8; do VSB_NO_SPLIT=1 $S --grid team=$t | sed 's/^{/{"no_split": 1, /' >> $O/sweep16.jsonl 2>>$O/sweep16.err; done
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest16.log 2>&1; echo "pytest rc=$?" >> $O/pytest16.log
echo done
