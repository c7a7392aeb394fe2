#!/bin/bash
# GPU tests after the staged-input spare-thread fix + bench line
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest14.log 2>&1; echo "pytest rc=$?" >> $O/pytest14.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke14.log 2>&1
timeout 900 python bench.py > $O/bench14.json 2> $O/bench14.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench14_ref.json 2> $O/bench14_ref.err
echo done
