#!/bin/bash
# round 2, run 12: grouped-team parity diagnosis (ldlt_57 team 8 x 2 groups, local search on)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 600 python tools/groups_diag.py ldlt_57 4096 '{"team": 8, "groups": 2}' > $O/r2_12_groups_rows.jsonl 2> $O/r2_12_groups_rows.err
VSB_LOCKSTEP=1 timeout 600 python tools/groups_diag.py ldlt_57 4096 '{"team": 8, "groups": 2}' > $O/r2_12_groups_rows_ls1.jsonl 2>> $O/r2_12_groups_rows.err
CS="timeout 1200 compute-sanitizer --print-limit 30"
$CS --tool racecheck python tools/sanitize_probe.py ldlt_57 128 '{"team": 8, "groups": 2}' > $O/r2_12_racecheck_ldlt57_g2.log 2>&1; echo "racecheck rc=$?"
$CS --tool synccheck python tools/sanitize_probe.py ldlt_57 128 '{"team": 8, "groups": 2}' > $O/r2_12_synccheck_ldlt57_g2.log 2>&1; echo "synccheck rc=$?"
$CS --tool memcheck python tools/sanitize_probe.py ldlt_57 128 '{"team": 8, "groups": 2}' > $O/r2_12_memcheck_ldlt57_g2.log 2>&1; echo "memcheck rc=$?"
$CS --tool initcheck python tools/sanitize_probe.py ldlt_57 128 '{"team": 8, "groups": 2}' > $O/r2_12_initcheck_ldlt57_g2.log 2>&1; echo "initcheck rc=$?"
