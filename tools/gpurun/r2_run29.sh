#!/bin/bash
# round 2, run 29: the whole GPU suite + smoke on the final tree (all workload plans prebuilt)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2_29_smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=10 > $O/r2_29_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2_29_pytest.log
