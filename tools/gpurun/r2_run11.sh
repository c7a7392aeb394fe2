#!/bin/bash
# round 2, run 11: shape sweeps of the small / mid thread-mode tapes at B=1e6 (occupancy,
# register caps, team mode for ldlt_12), ncu --set full of the five srbm_mpc chunks and of
# the small-tape tile kernels, sanitizer pass over the new paths (streamed inputs, constant
# table, local-search schedules, large-batch shape)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 20 --check 8"
D="timeout 900 python tools/sweep.py --steps 3 --check 256"
{
  # groups-mode parity diagnosis (run 10: ldlt_57 team 8 x 2 groups at B=65536 off by 4e-2)
  for E in "VSB_HC=1" "VSB_HC=0" "VSB_CONST_TABLE=0" "VSB_LOCKSTEP=1" "VSB_HC=0 VSB_CONST_TABLE=0 VSB_LOCKSTEP=1"; do
    $D --workload ldlt_57 --batch 4096 65536 --grid team=8 groups=2 --env $E
  done
  $D --workload ldlt_57 --batch 4096 65536 --grid team=8 groups=1
  $D --workload ldlt_57 --batch 65536 --grid team=12 groups=2
  $D --workload ldlt_25 --batch 65536 --grid team=8 groups=2
} > $O/r2_11_groups_diag.jsonl 2> $O/r2_11_groups_diag.err
echo "diag done"
timeout 3000 python -m pytest tests -m gpu -q -rf --junitxml=$O/r2_11_junit.xml > $O/r2_11_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 $O/r2_11_pytest.log
{
  $S --workload ldlt_12 --batch 1000000 --grid team=2,4,8
  $S --workload ldlt_12 --batch 1000000 --grid maxrregcount=96,128,168
  $S --workload ldlt_12 --batch 1000000 --grid bulk_io=-1 block=32,64,128
  $S --workload pendulum cartpole_rk4 --batch 1000000 --grid min_blocks=4,6,12,16
  $S --workload pendulum cartpole_rk4 --batch 1000000 --grid block=64,256
} > $O/r2_11_sweep.jsonl 2> $O/r2_11_sweep.err
echo "sweeps done"
R=/tmp/ncu_r2_11; mkdir -p $R
VSB_LINEINFO=1 timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"vsk_.*_c[0-9]+$" --launch-skip 5 --launch-count 5 \
  -o $R/srbm -f python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/r2_11_ncu_srbm.log 2>&1; echo "ncu srbm rc=$?"
ncu -i $R/srbm.ncu-rep --page raw --csv > $O/r2_11_ncu_srbm_raw.csv 2>/dev/null
for W in pendulum cartpole_rk4 ldlt_12; do
  VSB_LINEINFO=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"vsk_" --launch-skip 3 --launch-count 1 \
    -o $R/$W -f python tools/sweep.py --workload $W --batch 1000000 --steps 1 --warmup 1 > $O/r2_11_ncu_$W.log 2>&1; echo "ncu $W rc=$?"
  ncu -i $R/$W.ncu-rep --page raw --csv > $O/r2_11_ncu_${W}_raw.csv 2>/dev/null
done
CS="timeout 900 compute-sanitizer --print-limit 20"
for T in memcheck racecheck synccheck; do
  $CS --tool $T python tools/sanitize_probe.py srbm_mpc 64 > $O/r2_11_sanitize_${T}_srbm_t16.log 2>&1; echo "$T srbm rc=$?"
  $CS --tool $T python tools/sanitize_probe.py --host srbm_mpc 4096 > $O/r2_11_sanitize_${T}_srbm_host_stream_in.log 2>&1; echo "$T host rc=$?"
done
$CS --tool memcheck python tools/sanitize_probe.py srbm_mpc 20000 > $O/r2_11_sanitize_memcheck_srbm_wide.log 2>&1; echo "memcheck wide rc=$?"
$CS --tool synccheck python tools/sanitize_probe.py srbm_mpc 20000 > $O/r2_11_sanitize_synccheck_srbm_wide.log 2>&1; echo "synccheck wide rc=$?"
$CS --tool racecheck python tools/sanitize_probe.py humanoid_rbd 64 '{"flags": 0}' > $O/r2_11_sanitize_racecheck_humanoid.log 2>&1; echo "racecheck humanoid rc=$?"
du -sh $O
