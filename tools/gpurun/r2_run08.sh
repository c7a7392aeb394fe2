#!/bin/bash
# round 2, run 08: constant table (VSB_CONST_TABLE), schedule local search (VSB_HC), team width,
# barrier form -- A/B on the config workloads, all in one box session
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
MODE=${1:-run}
run() {  # env... -- sweep args
  if [ "$MODE" = compile ]; then python tools/sweep.py --compile-only "$@"; else timeout 900 python tools/sweep.py --steps 20 --check 8 "$@"; fi
}
for E in "VSB_HC=0 VSB_CONST_TABLE=0" "VSB_HC=0 VSB_CONST_TABLE=1" "VSB_HC=1 VSB_CONST_TABLE=1" "VSB_HC=1 VSB_CONST_TABLE=1 VSB_BAR_MBAR=0"; do
  run --workload srbm_mpc --batch 512 4096 65536 --grid team=12,16 --env $E
  run --workload humanoid_rbd ldlt_57 rbd_chain12 --batch 4096 65536 --env $E
done
for G in 0 64 256; do
  run --workload srbm_mpc --batch 65536 262144 --grid team=8 groups=2 --env VSB_HC=1 VSB_REMAT_GAP=$G
done
run --workload srbm_mpc --batch 262144 --grid team=12,16 --env VSB_HC=1
