#!/bin/bash
# DIVR opt-in test re-run; wide-I/O thread-mode tape (ldlt_12, 816 B/instance): block x TMA
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_divr.py -m gpu -q > $O/pytest66.log 2>&1; echo "rc=$?" >> $O/pytest66.log
timeout 900 python tools/sweep.py --steps 20 --workload ldlt_12 --batch 1000000 --check 8 --grid block=32,64,128 bulk_io=-1,1 > $O/sweep66.jsonl 2>$O/sweep66.err
timeout 900 python tools/sweep.py --steps 20 --workload ldlt_12 --batch 1000000 --check 8 --grid block=64 bulk_io=1 min_blocks=2,3,4 > $O/sweep66b.jsonl 2>>$O/sweep66.err
echo done
