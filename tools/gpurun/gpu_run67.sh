#!/bin/bash
# full GPU suite with the block-64 rule; ldlt_12 defaults across batches (fp64 / fp32)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest67.log 2>&1; echo "rc=$?" >> $O/pytest67.log
timeout 900 python tools/sweep.py --steps 20 --workload ldlt_12 --batch 4096 65536 1000000 --check 8 > $O/sweep67.jsonl 2>$O/sweep67.err
timeout 900 python tools/sweep.py --steps 20 --workload ldlt_12 --batch 4096 65536 1000000 --check 8 --dtype float32 >> $O/sweep67.jsonl 2>>$O/sweep67.err
echo done
