#!/bin/bash
# round 2, run 13: grouped-team parity vs the lockstep form (out-of-line call / inline / none)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
G='{"team": 8, "groups": 2}'
for E in "" "VSB_LOCKSTEP=1" "VSB_LS_INLINE=1"; do
  for W in "ldlt_57 4096" "srbm_mpc 20000" "srbm_mpc 4096"; do
    echo "== $E $W"
    env $E timeout 600 python tools/groups_diag.py $W "$G" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except ValueError: continue
    if d['bad_elems']: print(d['out'], d['bad_elems'], d['of'], d['max_err'])
print('done')"
  done
done > $O/r2_13_lockstep_forms.txt 2>&1
env timeout 600 python tools/groups_diag.py srbm_mpc 20000 > $O/r2_13_srbm_wide_default.jsonl 2>&1
VSB_LOCKSTEP=1 timeout 600 python tools/groups_diag.py srbm_mpc 20000 > $O/r2_13_srbm_wide_ls1.jsonl 2>&1
