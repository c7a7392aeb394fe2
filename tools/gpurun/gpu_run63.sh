#!/bin/bash
# full GPU suite + smoke + default bench line on the current tree
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest63.log 2>&1; echo "rc=$?" >> $O/pytest63.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke63.log 2>&1
timeout 900 python bench.py > $O/bench63.json 2> $O/bench63.err
echo done
