#!/bin/bash
# round 2, run 10: sorted warp-phase order after the local search, streamed H2D inputs for team
# plans (VSB_STREAM_IN), large-batch shape from 2 waves -- GPU suite, smoke, bench line, e2e A/B,
# launch list, libdevice-trig comparison of the small tapes
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -rf --junitxml=$O/r2_10_junit.xml > $O/r2_10_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 $O/r2_10_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_10_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/r2_10_bench.json 2> $O/r2_10_bench.err; echo "bench rc=$?"
for W in srbm_mpc humanoid_rbd; do for B in 4096 65536; do for S in 1 2 4 8; do
  VSB_STREAM_IN=$S timeout 300 python tools/e2e_probe.py --workload $W --batch $B >> $O/r2_10_e2e.jsonl 2>> $O/r2_10_e2e.err
done; done; done
VSB_TRACE=1 VSB_STREAM_IN=4 timeout 300 python tools/e2e_probe.py --workload srbm_mpc --batch 4096 --calls 3 > /dev/null 2> $O/r2_10_e2e_trace.txt
VSB_TRACE=1 VSB_STREAM_IN=1 timeout 300 python tools/e2e_probe.py --workload srbm_mpc --batch 4096 --calls 3 > /dev/null 2>> $O/r2_10_e2e_trace.txt
timeout 900 python tools/sweep.py --steps 20 --check 8 --workload pendulum cartpole_rk4 ldlt_12 --batch 1000000 --grid libdevice_trig=0,1 > $O/r2_10_sweep.jsonl 2> $O/r2_10_sweep.err
timeout 900 python tools/sweep.py --steps 20 --check 8 --workload humanoid_rbd --batch 16384 65536 --grid team=6,8,12 groups=2 >> $O/r2_10_sweep.jsonl 2>> $O/r2_10_sweep.err
timeout 900 python tools/sweep.py --steps 20 --check 8 --workload ldlt_57 rbd_chain12 --batch 65536 --grid team=8 groups=2 >> $O/r2_10_sweep.jsonl 2>> $O/r2_10_sweep.err
echo "sweeps done"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_10_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --no-numba > $O/r2_10_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
du -sh $O
