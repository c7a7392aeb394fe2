#!/bin/bash
# outlined DIV/trig subroutines + wave-filling instances per cluster
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc"
for spec in "team=12" "team=16" "team=8" "team=16 outline=-1" "team=12 outline=1"; do
  $S --batch 4096 --check 16 --grid $spec >> $O/sweep11.jsonl 2>>$O/sweep11.err
done
$S --batch 65536 --grid team=12 >> $O/sweep11.jsonl 2>>$O/sweep11.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest11.log 2>&1; echo "pytest rc=$?" >> $O/pytest11.log
echo done
