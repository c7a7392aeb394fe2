#!/bin/bash
# re-entry validation: full GPU test suite, smoke, default bench line
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest9.log 2>&1; echo "pytest rc=$?" >> $O/pytest9.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke9.log 2>&1
timeout 900 python bench.py > $O/bench9.json 2> $O/bench9.err
echo done
