#!/bin/bash
# round 2: team-barrier forms -- 0 barrier.sync (non-aligned, PTX-legal), 1 bar.sync 0, 2 named
# bar.sync 15, VS_BS -- timing + synccheck; lockstep x barrier form; acceptance fuzz (acc)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 20"
for m in 0 1 2; do
  $S --workload srbm_mpc humanoid_rbd --batch 4096 65536 --env VSB_BAR_ALIGNED=$m >> $O/r2_05_bar.jsonl 2>>$O/r2_05_bar.err
  $S --workload srbm_mpc humanoid_rbd --batch 4096 65536 --grid lockstep=2 --env VSB_BAR_ALIGNED=$m VSB_LOCKSTEP_EVERY=4 >> $O/r2_05_bar.jsonl 2>>$O/r2_05_bar.err
done
echo "bar done"
CS="timeout 900 compute-sanitizer --print-limit 10"
for m in 1 2; do
  VSB_BAR_ALIGNED=$m $CS --tool synccheck python tools/sanitize_probe.py srbm_mpc 64 > $O/r2_05_san_synccheck_srbm_mode$m.log 2>&1; echo "sync srbm mode $m rc=$?"
  VSB_BAR_ALIGNED=$m $CS --tool synccheck python tools/sanitize_probe.py humanoid_rbd 256 '{"team": 8, "lockstep": 4}' > $O/r2_05_san_synccheck_humanoid_lock_mode$m.log 2>&1; echo "sync humanoid mode $m rc=$?"
done
timeout 1800 python -m pytest "tests/test_acceptance_fuzz.py::test_acceptance_fuzz_gpu[acc]" -m gpu -x -q -rf > $O/r2_05_pytest_acc.log 2>&1; echo "pytest acc rc=$?"
grep -E "^E " $O/r2_05_pytest_acc.log | head -3 | cut -c1-400
echo "all done"
