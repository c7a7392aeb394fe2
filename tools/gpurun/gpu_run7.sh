#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 1200 python tools/sweep.py --steps 5 --warmup 2"
# config 4 scale: srbm at large batch, team variants (2 CTAs/SM candidates) and thread mode
$S --workload srbm_mpc --batch 65536 --grid team=4 team_smem=102400 > $O/sweep7.jsonl 2>&1
$S --workload srbm_mpc --batch 65536 --grid team=8 team_smem=102400 maxrregcount=128 >> $O/sweep7.jsonl 2>&1
$S --workload srbm_mpc --batch 65536 --grid team=1,12,16 >> $O/sweep7.jsonl 2>&1
# config 5: stress tapes fp64 + fp32 (error distribution vs the fp64 oracle)
$S --workload rbd_chain12 ldlt_57 --batch 4096 --check 64 >> $O/sweep7.jsonl 2>&1
$S --workload rbd_chain12 ldlt_57 --batch 4096 --check 64 --dtype float32 >> $O/sweep7.jsonl 2>&1
$S --workload rbd_chain12 ldlt_57 --batch 4096 --grid team=1 >> $O/sweep7.jsonl 2>&1
$S --workload srbm_mpc --batch 4096 --check 64 --dtype float32 >> $O/sweep7.jsonl 2>&1
$S --workload humanoid_rbd --batch 65536 --check 64 --dtype float32 --grid team=8 >> $O/sweep7.jsonl 2>&1
# config 4 proper: 1e6-instance global batch on 1 GPU
timeout 900 python bench.py --global-batch 1000000 --steps 3 --warmup 3 --cpu-seconds 5 > $O/bench7_1e6.json 2> $O/bench7_1e6.err
# DRAM traffic per kernel of one srbm step (for roofline.traffic)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:vsk_ --csv --log-file $O/traffic7_srbm.csv python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/ncu7.log 2>&1
echo done
