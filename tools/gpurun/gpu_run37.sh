#!/bin/bash
# instruction-cache evidence: ICC (per SM) / GCC (L1.5, per GPC) / L2 sectors from GCC, team chunk kernel
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
M=sm__icc_requests.sum,sm__icc_requests_lookup_hit.sum,sm__icc_requests_lookup_miss.sum,sm__icc_request_hit_rate.pct,gcc__cache_requests_type_instruction.sum,gcc__cache_requests_type_instruction_lookup_hit.sum,gcc__cache_requests_type_instruction_lookup_miss.sum,gcc__average_cache_request_type_instruction_hit_rate.pct,lts__t_sector_throughput_srcunit_gcc.pct,lts__average_t_sector_srcunit_gcc.ratio,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio
for b in 512 4096; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:vsk_ -c 5 --csv --log-file $O/icc37_srbm_$b.csv \
    python tools/sweep.py --workload srbm_mpc --batch $b --steps 1 --warmup 0 > /dev/null 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:vsk_ -c 1 --csv --log-file $O/icc37_cartpole.csv \
  python tools/sweep.py --workload cartpole_rk4 --batch 1000000 --steps 1 --warmup 0 > /dev/null 2>&1
echo done
