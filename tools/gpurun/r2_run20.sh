#!/bin/bash
# round 2, run 20: BatchPipeline (vsb_pipe_*) tests and the bench line with the pipelined e2e;
# L2 prefetch of chunk imports (VSB_SPREFETCH=D) and an L2 persisting window over the chunk
# scratch (VSB_L2_PERSIST_MB) on srbm_mpc B=4096, parity checked on 16 rows
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_contract.py -m gpu -q -x -rf -k pipeline > $O/r2_20_pytest_pipe.log 2>&1; echo "pipe tests rc=$?"
tail -2 $O/r2_20_pytest_pipe.log
timeout 900 python bench.py --no-secondary > $O/r2_20_bench.json 2> $O/r2_20_bench.err; echo "bench rc=$?"
S="timeout 900 python tools/sweep.py --steps 30 --check 16 --workload srbm_mpc --batch 4096"
{
  for rep in 1 2; do
    $S
    for d in 1 2 4; do VSB_SPREFETCH=$d $S | sed "s/^{/{\"spf\": $d, /"; done
    for m in 32 64 96; do VSB_TRACE=1 VSB_L2_PERSIST_MB=$m $S | sed "s/^{/{\"l2persist_mb\": $m, /"; done
    VSB_SPREFETCH=2 VSB_L2_PERSIST_MB=64 $S | sed "s/^{/{\"spf\": 2, \"l2persist_mb\": 64, /"
  done
} > $O/r2_20_sweep.jsonl 2> $O/r2_20_sweep.err

timeout 2700 python -m pytest tests -m gpu -q -x -rf > $O/r2_20_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2_20_pytest.log
