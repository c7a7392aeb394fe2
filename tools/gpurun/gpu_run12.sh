#!/bin/bash
# (1) is instruction fetch per-SM or chip-wide?  (2) groups at B=4096, with/without
# wave-filling ipc  (3) ncu --set full of one team chunk kernel
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python tools/ifetch_bench.py --scale --ops 6000 > $O/ifetch12.jsonl 2> $O/ifetch12.err
S="timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc"
for spec in "team=16" "team=12" "team=8 groups=2" "team=6 groups=2" "team=4 groups=4"; do
  $S --batch 4096 --check 16 --grid $spec >> $O/sweep12.jsonl 2>>$O/sweep12.err
  VSB_IPC_FILL=0 $S --batch 4096 --grid $spec | sed 's/^{/{"ipc_fill": 0, /' >> $O/sweep12.jsonl 2>>$O/sweep12.err
done
$S --batch 65536 --grid team=8 groups=2 >> $O/sweep12.jsonl 2>>$O/sweep12.err
$S --batch 65536 --grid team=12 >> $O/sweep12.jsonl 2>>$O/sweep12.err
for spec in "team=16" "team=16 groups=2 cluster=2"; do
  tag=$(echo $spec | tr -d ' =')
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:_c2 -c 1 -o $O/prof12_$tag \
    python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 --grid $spec > $O/ncu12_$tag.log 2>&1
done
echo done
