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

# (label, metric, wanted unit) -- values are converted from the unit row of the raw page
ROWS = [
    ("duration (us)", "gpu__time_duration.sum", "us"),
    ("DRAM read (MB)", "dram__bytes_read.sum", "MB"),
    ("DRAM write (MB)", "dram__bytes_write.sum", "MB"),
    ("DRAM throughput (% peak)", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("SM throughput (% peak)", "sm__throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("issue slots busy (%)", "sm__inst_issued.avg.pct_of_peak_sustained_active", ""),
    ("executed IPC (active)", "sm__inst_executed.avg.per_cycle_active", ""),
    ("instructions executed (M warp-instr)", "smsp__inst_executed.sum", "M"),
    ("achieved occupancy (%)", "sm__warps_active.avg.pct_of_peak_sustained_active", ""),
    ("registers / thread", "launch__registers_per_thread", ""),
    ("grid size", "launch__grid_size", ""),
    ("block size", "launch__block_size", ""),
    ("dynamic smem / block (KB)", "launch__shared_mem_per_block_dynamic", "KB"),
    ("local load sectors (M)", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "M"),
    ("local store sectors (M)", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "M"),
    ("global load sectors (M)", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "M"),
    ("global load requests (M)", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "M"),
    ("smem ld bank conflicts (M)", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "M"),
    ("smem st bank conflicts (M)", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "M"),
    ("L2 hit rate (%)", "lts__t_sector_hit_rate.pct", ""),
    ("FP64 pipe (% peak)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", ""),
]
STALL_PREFIX = "smsp__average_warps_issue_stalled_"
STALL_SUFFIX = "_per_issue_active.ratio"
_SCALE = {  # unit row -> factor to the base (bytes, seconds, count)
    "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3, "byte/block": 1,
    "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
}
_WANT = {"us": 1e-6, "MB": 1e6, "KB": 1e3, "M": 1e6}


def convert(value: float, unit: str, want: str) -> float:
    if not want:
        return value
    base = value * _SCALE.get(unit.strip(), 1.0)
    return base / _WANT[want]


def raw_rows(path):
    if path.endswith(".csv"):   # an `ncu -i ... --page raw --csv` export made on the GPU box
        with open(path) as fh:
            out = fh.read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
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
            for label, metric, want in ROWS:
                i = idx.get(metric)
                if i is None or not row[i].strip():
                    vals[label] = "-"
                    continue
                try:
                    vals[label] = f"{convert(float(row[i].replace(',', '')), units[i], want):.4g}"
                except ValueError:
                    vals[label] = row[i]
            stalls = []
            for h, i in idx.items():
                if h.startswith(STALL_PREFIX) and h.endswith(STALL_SUFFIX):
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
