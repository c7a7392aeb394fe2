#!/bin/bash
# host pipeline rework (H2D stream -> per-piece compute streams -> D2H stream); team_smem sweep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for pb in 4194304 2097152 1048576; do
  VSB_HOST_PIECE_BYTES=$pb timeout 300 python tools/e2e_probe.py >> $O/e2e23.jsonl 2>>$O/e2e23.err
done
VSB_HOST_PIECE_BYTES=4194304 timeout 300 python tools/e2e_probe.py --workload cartpole_rk4 --batch 1000000 >> $O/e2e23.jsonl 2>>$O/e2e23.err
timeout 600 python tools/sweep.py --steps 10 --workload srbm_mpc --batch 512 4096 --grid team=16 team_smem=65536,102400,153600,204800 > $O/sweep23.jsonl 2>$O/sweep23.err
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest23.log 2>&1; echo "pytest rc=$?" >> $O/pytest23.log
echo done
