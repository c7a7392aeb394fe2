#!/bin/bash
# round 2, run 07: mbarrier phase barriers + runtime lockstep flag + GVN + schedule local search
# (VSB_HC) -- barrier-form and HC A/B, per-phase clock64 timeline of the srbm_mpc /
# humanoid_rbd team chains (CTA 0)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 20"
for E in "VSB_HC=0 VSB_BAR_MBAR=1" "VSB_HC=1" "VSB_HC=0 VSB_BAR_MBAR=0" "VSB_HC=0 VSB_BAR_ALIGNED=1"; do
  $S --workload srbm_mpc --batch 512 4096 65536 --check 16 --env $E >> $O/r2_07_bar.jsonl 2>>$O/r2_07_bar.err
  $S --workload humanoid_rbd ldlt_57 rbd_chain12 --batch 4096 65536 --check 16 --env $E >> $O/r2_07_bar.jsonl 2>>$O/r2_07_bar.err
done
echo "sweep done"
for H in 0 1; do
  VSB_HC=$H VSB_CACHE_DIR=$PWD/.vsb_trace_cache timeout 600 python tools/phase_trace.py --workload srbm_mpc --batch 512 4096 > $O/r2_07_trace_srbm_hc$H.jsonl 2>> $O/r2_07_trace.err
done
VSB_HC=0 VSB_CACHE_DIR=$PWD/.vsb_trace_cache timeout 600 python tools/phase_trace.py --workload humanoid_rbd --batch 4096 65536 > $O/r2_07_trace_humanoid.jsonl 2>> $O/r2_07_trace.err
echo "trace done"
du -sh $O
