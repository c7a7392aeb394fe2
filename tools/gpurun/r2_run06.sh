#!/bin/bash
# round 2: defaults after the barrier / lockstep decisions -- sweep, full GPU suite, smoke,
# bench line, launch list, ncu --set full of the five srbm_mpc chunks (summarised on the box)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
S="timeout 900 python tools/sweep.py --steps 20"
$S --workload srbm_mpc humanoid_rbd ldlt_57 rbd_chain12 --batch 4096 65536 --grid lockstep=0,1 --check 8 > $O/r2_06_lock.jsonl 2>$O/r2_06_lock.err
for g in 64 256; do
  $S --workload srbm_mpc --batch 4096 65536 --check 8 --env VSB_REMAT_GAP=$g >> $O/r2_06_remat.jsonl 2>>$O/r2_06_remat.err
done
echo "sweep done"
timeout 2700 python -m pytest tests -m gpu -q -rf --junitxml=$O/r2_06_junit.xml > $O/r2_06_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 $O/r2_06_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_06_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2_06_bench.json 2> $O/r2_06_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_06_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_06_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
R=/tmp/ncu_r2_06; mkdir -p $R
VSB_LINEINFO=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"vsk_.*_c[0-9]+$" --launch-skip 5 --launch-count 5 \
  -o $R/srbm -f python tools/sweep.py --workload srbm_mpc --batch 4096 --steps 1 --warmup 1 > $O/r2_06_ncu_srbm.log 2>&1; echo "ncu srbm rc=$?"
python tools/ncu_summary.py $R/srbm.ncu-rep > $O/r2_06_ncu_srbm.md 2>>$O/r2_06_ncu_summary.err
ncu -i $R/srbm.ncu-rep --page raw --csv > $O/r2_06_ncu_srbm_raw.csv 2>/dev/null
du -sh $O
echo "all done"
