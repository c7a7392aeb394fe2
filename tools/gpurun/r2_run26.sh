#!/bin/bash
# round 2, run 26 (final tree: remat-128 one-wave shape, 24k-op chunks again for the large-batch
# shape): bench line, config 4, reference arm, the whole GPU suite with durations
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py > $O/r2_26_bench.json 2> $O/r2_26_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --global-batch 1000000 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_26_bench_config4.json 2> $O/r2_26_bench_config4.err; echo "bench config4 rc=$?"
timeout 600 python bench.py --impl reference > $O/r2_26_ref.json 2> $O/r2_26_ref.err; echo "ref rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2_26_smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -x -rf --durations=25 > $O/r2_26_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2_26_pytest.log
