#!/bin/bash
# trig fast path on/off x occupancy (thread mode), team-mode tapes, host pipeline piece size
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 600 python tools/sweep.py --steps 10"
for f in 1 0; do
  VSB_TRIG_FAST=$f $S --workload cartpole_rk4 pendulum --batch 1000000 --grid min_blocks=0,4,6,8 | sed "s/^{/{\"trig_fast\": $f, /" >> $O/sweep19.jsonl 2>>$O/sweep19.err
  VSB_TRIG_FAST=$f $S --workload humanoid_rbd --batch 4096 65536 | sed "s/^{/{\"trig_fast\": $f, /" >> $O/sweep19.jsonl 2>>$O/sweep19.err
  VSB_TRIG_FAST=$f $S --workload srbm_mpc --batch 4096 | sed "s/^{/{\"trig_fast\": $f, /" >> $O/sweep19.jsonl 2>>$O/sweep19.err
done
for pb in 4194304 2097152 1048576 524288; do
  VSB_HOST_PIECE_BYTES=$pb timeout 300 python tools/e2e_probe.py >> $O/e2e19.jsonl 2>>$O/e2e19.err
done
echo done
