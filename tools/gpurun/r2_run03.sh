#!/bin/bash
# round 2: non-aligned team barriers (A/B vs bar.sync), TMA pipeline depth sweep, GPU tests
# that failed in run 02, synccheck again, ncu --set full of the five srbm_mpc chunks and the
# cartpole / pendulum TMA kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 20"
$S --workload srbm_mpc --batch 4096 65536 --check 16 > $O/r2_03_bar.jsonl 2>$O/r2_03_bar.err
$S --workload srbm_mpc --batch 4096 65536 --env VSB_BAR_ALIGNED=1 >> $O/r2_03_bar.jsonl 2>>$O/r2_03_bar.err
$S --workload humanoid_rbd --batch 4096 65536 >> $O/r2_03_bar.jsonl 2>>$O/r2_03_bar.err
$S --workload humanoid_rbd --batch 4096 65536 --env VSB_BAR_ALIGNED=1 >> $O/r2_03_bar.jsonl 2>>$O/r2_03_bar.err
echo "bar done"
$S --workload pendulum cartpole_rk4 --batch 1000000 4000000 --grid bulk_io=1 tma_stages=2,3,4 block=128,256 --check 16 > $O/r2_03_tma.jsonl 2>$O/r2_03_tma.err
$S --workload pendulum cartpole_rk4 --batch 1000000 --grid bulk_io=1 tma_stages=3,4 min_blocks=4,6 >> $O/r2_03_tma.jsonl 2>>$O/r2_03_tma.err
echo "tma done"
timeout 1800 python -m pytest tests/test_acceptance_fuzz.py tests/test_gpu_contract.py "tests/test_gpu_parity.py::test_tma_tile_pipeline_equals_classic_kernel" -m gpu -q -rf > $O/r2_03_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2_03_pytest.log
CS="timeout 900 compute-sanitizer --print-limit 20"
$CS --tool synccheck python tools/sanitize_probe.py srbm_mpc 64 > $O/r2_03_san_synccheck_srbm_team16.log 2>&1; echo "sync srbm rc=$?"
$CS --tool synccheck python tools/sanitize_probe.py --fuzz acc 95 256 '{"team": 16, "team_smem": 2048}' > $O/r2_03_san_synccheck_fuzz_acc95_overflow.log 2>&1; echo "sync fuzz rc=$?"
$CS --tool synccheck python tools/sanitize_probe.py humanoid_rbd 64 '{"team": 8, "flags": 2}' > $O/r2_03_san_synccheck_humanoid_split.log 2>&1; echo "sync split rc=$?"
$CS --tool racecheck python tools/sanitize_probe.py humanoid_rbd 64 '{"team": 8, "flags": 3}' > $O/r2_03_san_racecheck_humanoid_pair_split.log 2>&1; echo "race pair+split rc=$?"
$CS --tool racecheck python tools/sanitize_probe.py pendulum 20000 '{"bulk_io": 1, "tma_stages": 4}' > $O/r2_03_san_racecheck_pendulum_tma4.log 2>&1; echo "race tma4 rc=$?"
export VSB_LINEINFO=1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"vsk_.*_c[0-9]+$" --launch-skip 5 --launch-count 5 \
  -o $O/r2_03_ncu_srbm -f python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/r2_03_ncu_srbm.log 2>&1; echo "ncu srbm rc=$?"
for w in cartpole_rk4 pendulum; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:_tma -c 1 -o $O/r2_03_ncu_$w -f \
  python tools/sweep.py --workload $w --batch 1000000 --steps 1 --warmup 1 > $O/r2_03_ncu_$w.log 2>&1; echo "ncu $w rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_03_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_03_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
for k in 1 2 3; do
  VSB_COPY_SPLIT=$k timeout 300 python tools/e2e_probe.py --workload srbm_mpc --batch 4096 --calls 20 > $O/r2_03_e2e_split$k.json 2>&1
done
echo "e2e done"
