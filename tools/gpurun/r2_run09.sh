#!/bin/bash
# round 2, run 09: new defaults (GVN, constant table, schedule local search, batch-adaptive
# large-batch shape) -- full GPU suite, smoke, bench line, launch list, sweeps of the schedule
# knobs and of the large-batch switch point
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
MODE=${1:-run}
run() {
  if [ "$MODE" = compile ]; then python tools/sweep.py --compile-only "$@"; else timeout 900 python tools/sweep.py --steps 20 --check 8 "$@"; fi
}
if [ "$MODE" = compile ]; then
  run --workload srbm_mpc --grid phase_cost=64,128,192 priority=0,1
  run --workload srbm_mpc --grid priority=1
  exit 0
fi
timeout 3000 python -m pytest tests -m gpu -q -rf -x --junitxml=$O/r2_09_junit.xml > $O/r2_09_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 $O/r2_09_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_09_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2_09_bench.json 2> $O/r2_09_bench.err; echo "bench rc=$?"
{
  run --workload srbm_mpc --batch 4096 --grid phase_cost=64,128,192 priority=0,1
  run --workload srbm_mpc --batch 512 4096 --grid priority=1
  for W in 0 9472 18944; do run --workload srbm_mpc --batch 16384 32768 65536 --env VSB_WIDE_MIN=$W; done
} > $O/r2_09_sweep.jsonl 2> $O/r2_09_sweep.err
echo "sweep done"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_09_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_09_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
du -sh $O
