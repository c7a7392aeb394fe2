#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/ifetch_bench.py --ops 6000 > $O/ifetch_reg.jsonl 2> $O/ifetch_reg.err
timeout 900 python tools/ifetch_bench.py --ops 6000 --consts > $O/ifetch_const.jsonl 2> $O/ifetch_const.err
echo done
