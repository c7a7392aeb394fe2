#!/bin/bash
# zero-copy outputs on the host path (kernels store into mapped pinned memory): e2e A/B + bitwise check
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for z in 0 1; do
  for w in "srbm_mpc 4096" "srbm_mpc 65536" "humanoid_rbd 4096" "pendulum 1000000" "cartpole_rk4 1000000" "ldlt_12 65536"; do
    set -- $w
    VSB_ZC_OUT=$z timeout 600 python tools/e2e_probe.py --workload $1 --batch $2 >> $O/e2e72.jsonl 2>>$O/e2e72.err
  done
done
done
echo done
