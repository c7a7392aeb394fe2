#!/bin/bash
# humanoid_rbd (config 2) at throughput batches: thread mode and narrow teams vs team 12
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 1500 python tools/sweep.py --steps 10 --workload humanoid_rbd --batch 65536 --check 8 --grid team=1,2,4,6,12 > $O/sweep73.jsonl 2>$O/sweep73.err
timeout 900 python tools/sweep.py --steps 10 --workload humanoid_rbd --batch 65536 --check 8 --grid team=1 chunk_ops=1500,3000,6000 > $O/sweep73b.jsonl 2>>$O/sweep73.err
echo done
