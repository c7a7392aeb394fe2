#!/bin/bash
# round 2, run 23 (final tree): bench line + reference arm, launch list of the bench command,
# ncu --set full of the five srbm_mpc chunks (remat 128 default), sanitizers on the new
# default and on the pipelined host path, the whole GPU suite
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py > $O/r2_23_bench.json 2> $O/r2_23_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/r2_23_ref.json 2> $O/r2_23_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_23_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_23_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
R=/tmp/ncu_r2_23; mkdir -p $R
VSB_LINEINFO=1 timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"vsk_.*_c[0-9]+$" --launch-skip 5 --launch-count 5 \
  -o $R/srbm -f python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/r2_23_ncu_srbm.log 2>&1; echo "ncu srbm rc=$?"
ncu -i $R/srbm.ncu-rep --page raw --csv > $O/r2_23_ncu_srbm_raw.csv 2>/dev/null
CS="timeout 900 compute-sanitizer --print-limit 20"
for T in memcheck racecheck synccheck; do
  $CS --tool $T python tools/sanitize_probe.py srbm_mpc 64 > $O/r2_23_sanitize_${T}_srbm_t16_remat.log 2>&1; echo "$T srbm rc=$?"
done
$CS --tool memcheck python tools/sanitize_probe.py --pipe srbm_mpc 4096 > $O/r2_23_sanitize_memcheck_pipe.log 2>&1; echo "memcheck pipe rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -x -rf > $O/r2_23_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/r2_23_pytest.log
