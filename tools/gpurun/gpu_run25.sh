#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for pb in 16777216 4194304 1048576; do
  VSB_TRACE=1 VSB_HOST_PIECE_BYTES=$pb timeout 300 python tools/e2e_probe.py --calls 5 > $O/e2e25_$pb.out 2> $O/e2e25_$pb.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > $O/bench25_torchrun.json 2> $O/bench25_torchrun.err
echo done
