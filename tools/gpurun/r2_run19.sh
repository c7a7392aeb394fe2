#!/bin/bash
# round 2, run 19 (fresh container re-entry): the whole GPU suite, smoke, the default bench
# line, the reference arm and the launch list of the bench command
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r2_19_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2_19_bench.json 2> $O/r2_19_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/r2_19_ref.json 2> $O/r2_19_ref.err; echo "ref rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -x -rf > $O/r2_19_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2_19_pytest.log
