#!/usr/bin/env python
"""Summarise `ncu --set full` reports as a markdown table (runs here, on the
.ncu-rep files gpurun brings back):

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [more.ncu-rep ...] > profiles/r2_ncu_x.md

One column per profiled launch: duration, DRAM bytes and throughput, SM / issue
activity, occupancy, registers, local-memory (spill) traffic, shared-memory bank
conflicts, the top warp-stall reasons (cycles per issued instruction) and the
executed-instruction mix by SASS opcode class.
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

ROWS = [
    ("duration (us)", "gpu__time_duration.sum", 1e-3),
    ("DRAM read (MB)", "dram__bytes_read.sum", 1e-6),
    ("DRAM write (MB)", "dram__bytes_write.sum", 1e-6),
    ("DRAM throughput (% peak)", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("SM throughput (% peak)", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue slots busy (%)", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("executed IPC (active)", "sm__inst_executed.avg.per_cycle_active", 1),
    ("instructions executed (M warp-instr)", "smsp__inst_executed.sum", 1e-6),
    ("achieved occupancy (%)", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("registers / thread", "launch__registers_per_thread", 1),
    ("grid size", "launch__grid_size", 1),
    ("block size", "launch__block_size", 1),
    ("dynamic smem / block (KB)", "launch__shared_mem_per_block_dynamic", 1e-3),
    ("local load sectors (M)", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", 1e-6),
    ("local store sectors (M)", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", 1e-6),
    ("smem ld bank conflicts (M)", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1e-6),
    ("smem st bank conflicts (M)", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", 1e-6),
    ("L2 hit rate (%)", "lts__t_sector_hit_rate.pct", 1),
    ("FP64 pipe (% peak)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("FP64 instr executed (M)", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 1e-6 / 32),
]
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"
STALL_SUFFIX = ".ratio"
MIX_PREFIX = "sass__inst_executed_per_opcode"


def raw_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units, data = rows[0], rows[1], rows[2:]
    return header, units, data


def main():
    cols = []
    for path in sys.argv[1:]:
        header, units, data = raw_rows(path)
        idx = {h: i for i, h in enumerate(header)}
        for row in data:
            name = row[idx.get("Kernel Name", 0)][:48]
            vals = {}
            for label, metric, scale in ROWS:
                i = idx.get(metric)
                if i is None or not row[i].strip():
                    vals[label] = "-"
                    continue
                try:
                    vals[label] = f"{float(row[i].replace(',', '')) * scale:.4g}"
                except ValueError:
                    vals[label] = row[i]
            stalls = []
            for h, i in idx.items():
                if h.startswith(STALL_PREFIX) and h.endswith(STALL_SUFFIX) and "not_issued" not in h:
                    try:
                        stalls.append((float(row[i].replace(',', '')), h[len(STALL_PREFIX):-len(STALL_SUFFIX)]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            vals["top stalls (cycles / issued instr)"] = ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5])
            cols.append((f"{path.split('/')[-1]}: {name}", vals))
    if not cols:
        return
    labels = [r[0] for r in ROWS] + ["top stalls (cycles / issued instr)"]
    print("| metric | " + " | ".join(c[0] for c in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for lab in labels:
        print(f"| {lab} | " + " | ".join(c[1].get(lab, "-") for c in cols) + " |")


if __name__ == "__main__":
    main()
