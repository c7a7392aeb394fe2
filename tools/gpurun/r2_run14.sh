#!/bin/bash
# round 2, run 14: bitwise parity of srbm_mpc at B=20000 across shapes (the grouped large-batch
# variant showed a 3.5e-18 deviation), ldlt_57 grouped without lockstep; timing of the grouped
# variant without lockstep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
m() {  # label, env..., -- args
  python -c "
import json, sys
m = 0.0; bad = 0
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except ValueError: continue
    m = max(m, d['max_err']); bad += d['bad_elems']
print(sys.argv[2], 'max_err', m, 'bad', bad)" /tmp/gd.jsonl "$1"
}
run() { label=$1; shift; env "$@" > /tmp/gd.jsonl 2>&1; m "$label"; }
{
run "srbm 20000 team16 (no wide)" VSB_WIDE_MIN=0 timeout 600 python tools/groups_diag.py srbm_mpc 20000
run "srbm 20000 wide default" timeout 600 python tools/groups_diag.py srbm_mpc 20000
run "srbm 20000 wide HC=0" VSB_HC=0 timeout 600 python tools/groups_diag.py srbm_mpc 20000
run "srbm 20000 wide remat0" VSB_REMAT_GAP=0 timeout 600 python tools/groups_diag.py srbm_mpc 20000
run "srbm 20000 wide ls1" VSB_LOCKSTEP=1 timeout 600 python tools/groups_diag.py srbm_mpc 20000
run "srbm 4096 t8g2" timeout 600 python tools/groups_diag.py srbm_mpc 4096 '{"team": 8, "groups": 2}'
run "srbm 4096 t8g1" timeout 600 python tools/groups_diag.py srbm_mpc 4096 '{"team": 8}'
run "srbm 4096 t16" timeout 600 python tools/groups_diag.py srbm_mpc 4096
run "ldlt57 4096 t8g2 ls1" VSB_LOCKSTEP=1 timeout 600 python tools/groups_diag.py ldlt_57 4096 '{"team": 8, "groups": 2}'
run "ldlt57 4096 t12 default" timeout 600 python tools/groups_diag.py ldlt_57 4096
} > $O/r2_14_bitwise.txt 2>&1
timeout 900 python tools/sweep.py --steps 20 --check 8 --workload srbm_mpc --batch 16384 65536 --env VSB_LOCKSTEP=1 > $O/r2_14_sweep.jsonl 2> $O/r2_14_sweep.err
timeout 900 python tools/sweep.py --steps 20 --check 8 --workload srbm_mpc --batch 16384 65536 >> $O/r2_14_sweep.jsonl 2>> $O/r2_14_sweep.err
