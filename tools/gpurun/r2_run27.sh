#!/bin/bash
# round 2, run 27: BatchPipeline depth 1/2/3 vs synchronous batch_eval, e2e, per workload
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
{
  timeout 300 python tools/pipe_probe.py srbm_mpc 4096
  timeout 300 python tools/pipe_probe.py humanoid_rbd 4096
  timeout 300 python tools/pipe_probe.py humanoid_rbd 65536
  timeout 300 python tools/pipe_probe.py cartpole_rk4 1000000
  timeout 300 python tools/pipe_probe.py srbm_mpc 65536 --steps 10
} > $O/r2_27_pipe.jsonl 2> $O/r2_27_pipe.err
