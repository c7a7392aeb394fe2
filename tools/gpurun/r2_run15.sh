#!/bin/bash
# round 2, run 15: round-2 defaults as committed -- full GPU suite, smoke, bench line (default
# and config 4 at 1e6), launch list, the large-batch shape with and without lockstep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -rf --junitxml=$O/r2_15_junit.xml > $O/r2_15_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 $O/r2_15_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_15_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2_15_bench.json 2> $O/r2_15_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --global-batch 1000000 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_15_bench_config4.json 2> $O/r2_15_bench_config4.err; echo "bench config4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_15_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_15_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
du -sh $O
