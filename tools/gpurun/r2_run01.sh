#!/bin/bash
# round 2 baseline: full GPU suite, smoke, default bench line
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r2_01_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r2_01_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_01_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/r2_01_bench.json 2>$O/r2_01_bench.err; echo "bench rc=$?"
tail -3 $O/r2_01_pytest.log
