#!/usr/bin/env python
"""Join a phase timeline (tools/phase_trace.py, GPU) with the scheduler's per-warp phase loads
(tools/sched_probe, CPU) and summarise where the cycles of a team kernel chain go.

    python tools/phase_trace_report.py gpurun_out/r2_07_trace_srbm_hc0.jsonl [--hc 0]

Per chunk: cycles, phases, cycles per phase, and a least-squares fit of each phase's duration
against the phase's maximum warp load (cost units) -- cycles per unit on the critical warp and a
fixed per-phase cost (barrier + ramp) -- plus the share of the duration the busiest warp was busy.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sched_loads(workload: str, team: int, hc: int) -> list[np.ndarray]:
    """Per chunk: array [P, W] of scheduled cost units (VSB_SCHED_LOADS from the probe)."""
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sched_probe.py"), workload, str(team)],
                   check=True, capture_output=True)
    env = dict(os.environ, VSB_SCHED_LOADS="1", VSB_HC=str(hc))
    r = subprocess.run(["/tmp/vsb_sched_probe", f"/tmp/vsb_{workload}.bin", str(team)], env=env,
                       capture_output=True, text=True, check=True)
    chunks, cur = [], []
    for line in r.stderr.splitlines():
        if not line.startswith("loads "):
            continue
        head, vals = line.split(":", 1)
        ph = int(head.split()[1])
        if ph == 0 and cur:
            chunks.append(np.array(cur))
            cur = []
        cur.append([float(x) for x in vals.split()])
    if cur:
        chunks.append(np.array(cur))
    return chunks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--hc", type=int, default=None, help="VSB_HC of the traced plan (default: from the file name)")
    args = ap.parse_args()
    hc = args.hc if args.hc is not None else (1 if "hc1" in os.path.basename(args.trace) else 0)
    recs = [json.loads(line) for line in open(args.trace) if line.strip()]
    loads = None
    for r in recs:
        if loads is None:
            loads = sched_loads(r["workload"], r["W"], hc)
        arr, dep = np.array(r["arrive"], dtype=np.float64), np.array(r["depart"], dtype=np.float64)
        P, W = arr.shape
        ld = loads[r["chunk"]] if r["chunk"] < len(loads) else None
        rel = np.empty(P)   # barrier release of phase p (= earliest departure)
        rel[:-1] = dep[:-1].min(axis=1)
        rel[-1] = arr[-1].max()
        start = np.array(r["start"], dtype=np.float64)
        prev = np.concatenate([[start.min()], rel[:-1]])
        dur = rel - prev
        prev_w = np.vstack([start[None, :], dep[:-1]])
        busy = arr - prev_w                      # per warp time until it reached the barrier
        out = {"batch": r["batch"], "chunk": r["chunk"], "W": W, "P": P, "cycles": float(rel[-1] - start.min()),
               "cycles_per_phase": float(dur.mean())}
        if ld is not None and ld.shape == (P, W):
            mx = ld.max(axis=1)
            A = np.vstack([mx, np.ones(P)]).T
            coef, *_ = np.linalg.lstsq(A, dur, rcond=None)
            crit = ld.argmax(axis=1)
            crit_busy = busy[np.arange(P), crit]
            out.update({"fit_cycles_per_unit": float(coef[0]), "fit_cycles_per_phase": float(coef[1]),
                        "r2": float(1 - ((A @ coef - dur) ** 2).sum() / ((dur - dur.mean()) ** 2).sum()),
                        "sum_max_load": float(mx.sum()), "cycles_per_max_unit": float(dur.sum() / mx.sum()),
                        "crit_busy_share": float(crit_busy.sum() / dur.sum()),
                        "total_units": float(ld.sum())})
        else:
            out["loads"] = "schedule mismatch" if ld is not None else "none"
            if ld is not None:
                out["sched_shape"] = list(ld.shape)
        print(json.dumps(out))


if __name__ == "__main__":
    main()
