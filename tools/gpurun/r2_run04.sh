#!/bin/bash
# round 2 (re-run of 03, whose gpurun_out exceeded the 64 MiB pull limit: ncu reports are now
# summarised on the box and deleted) + lockstep-cluster sweep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 20"
$S --workload srbm_mpc --batch 4096 65536 --check 16 > $O/r2_04_bar.jsonl 2>$O/r2_04_bar.err
$S --workload srbm_mpc --batch 4096 65536 --env VSB_BAR_ALIGNED=1 >> $O/r2_04_bar.jsonl 2>>$O/r2_04_bar.err
$S --workload humanoid_rbd --batch 4096 65536 >> $O/r2_04_bar.jsonl 2>>$O/r2_04_bar.err
$S --workload humanoid_rbd --batch 4096 65536 --env VSB_BAR_ALIGNED=1 >> $O/r2_04_bar.jsonl 2>>$O/r2_04_bar.err
echo "bar done"
for E in 4 8 16; do
  $S --workload srbm_mpc humanoid_rbd --batch 4096 65536 --grid lockstep=2,4,8 --check 8 --env VSB_LOCKSTEP_EVERY=$E >> $O/r2_04_lock.jsonl 2>>$O/r2_04_lock.err
done
echo "lock done"
$S --workload pendulum cartpole_rk4 --batch 1000000 4000000 --grid bulk_io=1 tma_stages=2,3,4 block=128,256 --check 16 > $O/r2_04_tma.jsonl 2>$O/r2_04_tma.err
$S --workload pendulum cartpole_rk4 --batch 1000000 --grid bulk_io=1 tma_stages=3,4 min_blocks=4,6 >> $O/r2_04_tma.jsonl 2>>$O/r2_04_tma.err
echo "tma done"
timeout 1800 python -m pytest "tests/test_acceptance_fuzz.py::test_acceptance_fuzz_gpu[acc]" -m gpu -x -q -rf > $O/r2_04_pytest_acc.log 2>&1; echo "pytest acc rc=$?"
grep -m3 "Error" $O/r2_04_pytest_acc.log
CS="timeout 900 compute-sanitizer --print-limit 10"
$CS --tool synccheck python tools/sanitize_probe.py srbm_mpc 64 > $O/r2_04_san_synccheck_srbm_team16.log 2>&1; echo "sync srbm rc=$?"
$CS --tool synccheck python tools/sanitize_probe.py --fuzz acc 95 256 '{"team": 16, "team_smem": 2048}' > $O/r2_04_san_synccheck_fuzz_acc95_overflow.log 2>&1; echo "sync fuzz rc=$?"
$CS --tool synccheck python tools/sanitize_probe.py humanoid_rbd 64 '{"team": 8, "flags": 2}' > $O/r2_04_san_synccheck_humanoid_split.log 2>&1; echo "sync split rc=$?"
$CS --tool racecheck python tools/sanitize_probe.py humanoid_rbd 64 '{"team": 8, "flags": 3}' > $O/r2_04_san_racecheck_humanoid_pair_split.log 2>&1; echo "race pair+split rc=$?"
$CS --tool racecheck python tools/sanitize_probe.py pendulum 20000 '{"bulk_io": 1, "tma_stages": 4}' > $O/r2_04_san_racecheck_pendulum_tma4.log 2>&1; echo "race tma4 rc=$?"
$CS --tool synccheck python tools/sanitize_probe.py humanoid_rbd 256 '{"team": 8, "lockstep": 4}' > $O/r2_04_san_synccheck_humanoid_lockstep.log 2>&1; echo "sync lockstep rc=$?"
for k in 1 2 3; do
  VSB_COPY_SPLIT=$k timeout 300 python tools/e2e_probe.py --workload srbm_mpc --batch 4096 --calls 20 > $O/r2_04_e2e_split$k.json 2>&1
done
echo "e2e done"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_04_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_04_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
export VSB_LINEINFO=1
R=/tmp/ncu_r2_04; mkdir -p $R
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"vsk_.*_c[0-9]+$" --launch-skip 5 --launch-count 5 \
  -o $R/srbm -f python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/r2_04_ncu_srbm.log 2>&1; echo "ncu srbm rc=$?"
for w in cartpole_rk4 pendulum; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:_tma -c 1 -o $R/$w -f \
  python tools/sweep.py --workload $w --batch 1000000 --steps 1 --warmup 1 > $O/r2_04_ncu_$w.log 2>&1; echo "ncu $w rc=$?"
done
for r in srbm cartpole_rk4 pendulum; do
  python tools/ncu_summary.py $R/$r.ncu-rep > $O/r2_04_ncu_$r.md 2>>$O/r2_04_ncu_summary.err
  ncu -i $R/$r.ncu-rep --page raw --csv > $O/r2_04_ncu_${r}_raw.csv 2>/dev/null
  ncu -i $R/$r.ncu-rep --page details --csv > $O/r2_04_ncu_${r}_details.csv 2>/dev/null
done
du -sh $O
echo "all done"
