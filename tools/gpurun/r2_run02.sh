#!/bin/bash
# round 2: full GPU suite (acceptance fuzz, config-batch contract, fp32 per config, variants),
# fp32 error probe, compute-sanitizer logs, e2e timeline probe, default bench line
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf --junitxml=$O/r2_02_junit.xml > $O/r2_02_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 $O/r2_02_pytest.log
timeout 600 python tools/fp32_probe.py > $O/r2_02_fp32.jsonl 2> $O/r2_02_fp32.err; echo "fp32 rc=$?"
CS="timeout 900 compute-sanitizer --print-limit 20"
for tool in memcheck racecheck synccheck; do
  $CS --tool $tool python tools/sanitize_probe.py srbm_mpc 64 > $O/r2_02_san_${tool}_srbm_team16.log 2>&1; echo "san $tool srbm rc=$?"
  $CS --tool $tool python tools/sanitize_probe.py pendulum 20000 '{"bulk_io": 1}' > $O/r2_02_san_${tool}_pendulum_tma.log 2>&1; echo "san $tool tma rc=$?"
  $CS --tool $tool python tools/sanitize_probe.py --fuzz acc 95 256 '{"team": 16, "team_smem": 2048}' > $O/r2_02_san_${tool}_fuzz_acc95_overflow.log 2>&1; echo "san $tool fuzz rc=$?"
done
for pb in 0 2000000 4000000; do
  if [ $pb = 0 ]; then VSB_TRACE=1 timeout 300 python tools/e2e_probe.py --workload srbm_mpc --batch 4096 --calls 10 > $O/r2_02_e2e_p$pb.json 2> $O/r2_02_e2e_p$pb.err;
  else VSB_TRACE=1 VSB_HOST_PIECE_BYTES=$pb timeout 300 python tools/e2e_probe.py --workload srbm_mpc --batch 4096 --calls 10 > $O/r2_02_e2e_p$pb.json 2> $O/r2_02_e2e_p$pb.err; fi
done
timeout 900 python bench.py > $O/r2_02_bench.json 2> $O/r2_02_bench.err; echo "bench rc=$?"
