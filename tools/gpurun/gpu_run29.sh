#!/bin/bash
# full validation of the current tree: GPU suite, smoke, bench line, reference arm, launch list
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest29.log 2>&1; echo "pytest rc=$?" >> $O/pytest29.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke29.log 2>&1
timeout 900 python bench.py > $O/bench29.json 2> $O/bench29.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench29_ref.json 2> $O/bench29_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches29.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > $O/ncu29_launch.log 2>&1
echo done
