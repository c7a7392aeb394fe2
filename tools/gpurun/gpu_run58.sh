#!/bin/bash
# upper bound of DIV's share of the step: DIV rows rewritten to MUL (timing only)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python tools/op_probe.py --workload srbm_mpc --batch 4096 65536 --swap DIV=MUL > $O/probe58.jsonl 2>$O/probe58.err
timeout 600 python tools/op_probe.py --workload ldlt_57 --batch 4096 --swap DIV=MUL >> $O/probe58.jsonl 2>>$O/probe58.err
echo done
