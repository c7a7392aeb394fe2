#!/bin/bash
# round-final record: full GPU suite, smoke, bench line (N=1 default), reference arm, launch list
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest75.log 2>&1; echo "rc=$?" >> $O/pytest75.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke75.log 2>&1
timeout 900 python bench.py > $O/bench75.json 2> $O/bench75.err
timeout 900 python bench.py --impl reference > $O/bench75_ref.json 2> $O/bench75_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches75.csv python bench.py --steps 2 --warmup 3 --no-secondary > $O/ncu75.log 2>&1
echo done
