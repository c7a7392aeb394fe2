#!/bin/bash
# round 2, run 28: the default bench line with the depth-3 pipelined e2e
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py > $O/r2_28_bench.json 2> $O/r2_28_bench.err; echo "bench rc=$?"
timeout 600 python -m pytest tests/test_gpu_contract.py -m gpu -q -x -k pipeline > $O/r2_28_pytest_pipe.log 2>&1; echo "pipe tests rc=$?"
