#!/bin/bash
# full GPU suite + smoke on the final tree
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest81.log 2>&1; echo "rc=$?" >> $O/pytest81.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke81.log 2>&1
echo done
