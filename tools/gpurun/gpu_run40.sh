#!/bin/bash
# duplicate one-instruction operands instead of waiting a phase (VSB_DUP) -- A/B + team parity
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10"
for d in 1 0; do
  export VSB_DUP=$d
  $S --workload srbm_mpc --batch 512 4096 --check 16 | sed "s/^{/{\"dup\": $d, /" >> $O/sweep40.jsonl 2>>$O/sweep40.err
  $S --workload humanoid_rbd --batch 4096 65536 --check 16 | sed "s/^{/{\"dup\": $d, /" >> $O/sweep40.jsonl 2>>$O/sweep40.err
  $S --workload ldlt_57 --batch 4096 --check 16 | sed "s/^{/{\"dup\": $d, /" >> $O/sweep40.jsonl 2>>$O/sweep40.err
done
unset VSB_DUP
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "team or srbm or serial or shuffling or workloads" > $O/pytest40.log 2>&1; echo "rc=$?" >> $O/pytest40.log
echo done
