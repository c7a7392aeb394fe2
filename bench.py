#!/usr/bin/env python
"""Benchmark: batched tape evaluation on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload srbm_mpc] [--batch 4096]

One *step* = one evaluation of the workload's tape for the whole per-rank
batch (default: the MIT-Humanoid closed-form-MPC surrogate ``srbm_mpc``,
111,646 rows, batch 4096 per GPU -- BASELINE.json configs[2], the config the
north-star target is quoted on).  Inputs are resident in HBM; L2 is flushed
(256 MiB write) before every timed step, outside the timed events.
``value`` = evaluations/s over all ranks (CUDA events on the launch stream,
max over ranks).  ``e2e`` = the same metric through the reference-shaped
public API ``batch_eval(tape, BatchWorkspace)`` with pinned host buffers:
H2D of the inputs, the kernels and D2H of the outputs every step.
``cpu_baseline`` = the CPU oracle (a C restatement of the reference's
``run_range``/``batch_eval``) on the box's host cores, rank 0, N=1 only.
``--impl reference`` times that CPU path alone (rank 0; other ranks exit 0).

Multi-GPU: one process per GPU under torchrun; each rank evaluates its own
``--batch`` instances (weak scaling, no collective on the data path); the
only collectives are the timing barrier and a MAX all-reduce of the
elapsed time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("VSB_CACHE_DIR", os.path.join(ROOT, ".vsb_cache"))

METRIC = "function evals/sec (fp64) at batch 1e2–1e6 on 1/2/4/8 B200 vs CPU ref; % HBM roofline"
WORKLOAD_CONFIG = {
    "srbm_mpc": "MIT Humanoid closed-form MPC (fixed-iteration unrolled solver as one SX function) batch 4096 on 1 B200"
                " [surrogate: SRBM penalty-SQP T=6 M=1 M_inner=2, 111,646-row tape]",
    "cartpole_rk4": "cartpole/pendulum RK4 dynamics step casadi SX function, batch 1000, fp64",
    "humanoid_rbd": "MIT Humanoid rigid-body dynamics (mass matrix + bias forces) [surrogate: 24-DOF CRBA+RNEA]",
    "rbd_chain12": "large-tape stress: Lagrangian + symbolic-AD 12-link chain (>1e5 rows)",
    "ldlt_57": "large-tape stress: symbolic LDL^T solve n=57 (>1e5 rows)",
}


def arm_config(args, world: int, tape) -> dict:
    """The workload description both arms print (identical dicts: the driver compares them)."""
    per_gpu = args.global_batch // max(world, 1) if args.global_batch else args.batch
    total = args.global_batch if args.global_batch else args.batch * max(world, 1)
    return {"workload": args.workload, "batch_per_gpu": per_gpu, "global_batch": total,
            "description": WORKLOAD_CONFIG.get(args.workload, ""), "tape_rows": tape.n_instructions,
            "parallelism": f"batch-sharded x{world} (no data-path collective)"}


REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def reference_numba(tape, inputs, threads: int, seconds: float = 3.0):
    """The reference evaluator itself (numba ``run_range`` under ``vecsym.batchrt.batch_eval``,
    batchrt.py:194-244, _kernels.py:54-206) from ``baseline/_ref`` on the host cores:
    evals/s at W=1 and W=threads on bounded samples (2 warm-ups -- the first JITs --
    then the median of >= 5 calls and >= `seconds` of work, the reference's bench.py:133-156
    protocol).  None when the reference is not installed."""
    if not os.path.isdir(os.path.join(REF_PATH, "vecsym")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/vsb_numba_cache")
    if REF_PATH not in sys.path:
        sys.path.append(REF_PATH)
    try:
        from vecsym.batchrt import BatchWorkspace as RefWorkspace
        from vecsym.batchrt import batch_eval as ref_batch_eval
        from vecsym.tape import deserialize as ref_deserialize

        from paper_2408_09662_b200.tape import serialize
    except Exception as e:  # noqa: BLE001
        return {"error": f"import: {e}"[:200]}
    rtape = ref_deserialize(serialize(tape))
    res = {"kind": "reference", "impl": "vecsym.batchrt.batch_eval (numba run_range), baseline/_ref",
           "unit": "evals/s"}
    for w in (1, threads):
        B = max(w, min(inputs[0].shape[0], int(0.25 * w / max(tape.n_instructions * 4.5e-9, 1e-12))))
        ws = RefWorkspace(rtape, B)
        for i, v in enumerate(inputs):
            ws.set_input(i, v[:B])
        for _ in range(2):
            ref_batch_eval(rtape, ws, n_threads=w)
        rates, t_all = [], time.perf_counter()
        while len(rates) < 5 or (time.perf_counter() - t_all < seconds and len(rates) < 100):
            t0 = time.perf_counter()
            ref_batch_eval(rtape, ws, n_threads=w)
            rates.append(B / (time.perf_counter() - t0))
        res[f"w{w}" if w == 1 else "w_all"] = statistics.median(rates)
        res[f"sample_w{w}" if w == 1 else "sample_w_all"] = f"{B} instances x {len(rates)} calls"
    res["cores"] = threads
    return res


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = []
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8 or not f[0].isdigit() or int(f[0]) != self.gpu:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), f[4:8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, r in rows for k in range(4) if r[k].lower() == "active"})
        busy = [s for s, _, _ in rows if s > 0.5 * rows[0][1]] or [s for s, _, _ in rows]
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(m for _, m, _ in rows),
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline(tape, inputs, seconds: float, threads: int):
    """Oracle port on host cores: 2 warm-ups, then >= 5 reps and >= `seconds`
    of work; median evals/s (mirrors bench.py:133-156 of the reference)."""
    import oracle

    B = inputs[0].shape[0]
    ws = oracle.Workspace(tape, B)
    ws.set_inputs(inputs)
    for _ in range(2):
        ws.run(threads)
    rates, t_all = [], time.perf_counter()
    while len(rates) < 5 or time.perf_counter() - t_all < seconds:
        t0 = time.perf_counter()
        ws.run(threads)
        rates.append(B / (time.perf_counter() - t0))
        if len(rates) >= 200:
            break
    return statistics.median(rates), len(rates), time.perf_counter() - t_all


def cpu_sample_batch(tape, B: int, threads: int) -> int:
    """Largest sample <= B that keeps one oracle call under ~2 s (est. 4.5 ns/row-op/core)."""
    per_eval = tape.n_instructions * 4.5e-9 / max(1, threads)
    cap = max(threads, int(2.0 / max(per_eval, 1e-12)))
    return int(min(B, cap))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import workloads

    tape = workloads.load_tape(args.workload)
    threads = len(os.sched_getaffinity(0))
    Bs = cpu_sample_batch(tape, args.batch, threads)
    inputs = workloads.make_inputs(args.workload, Bs, seed=0)
    import oracle

    ws = oracle.Workspace(tape, Bs)
    ws.set_inputs(inputs)
    for _ in range(max(args.warmup, 0)):
        ws.run(threads)
    # and at least 1 s of work, so that page faults of the work arrays and the host cores'
    # clock ramp are not timed (a 3-step run otherwise reads ~2x low)
    t_warm = time.perf_counter()
    while time.perf_counter() - t_warm < 1.0:
        ws.run(threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ws.run(threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = Bs * args.steps / total
    numba = reference_numba(tape, inputs, threads) if not args.no_numba else None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.global_batch else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": arm_config(args, args.gpus, tape),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "sample": f"{Bs} of {args.batch} instances per step, {args.steps} steps, "
                                   "oracle/vs_oracle.c (C restatement of vecsym run_range/batch_eval), pthreads",
                         "reference_numba": numba},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def issue_roof(workload, B, mean_s, clocks):
    """Instruction-issue view of the team kernels.

    Warp-instructions executed per step come from the committed ncu capture of the same
    plan (profiles/traffic.json <- r2_ncu_srbm_chunks_run11_raw.csv); divided by the live
    step time they give the chip's issue rate, against 148 SMs x 4 schedulers x clock.  A
    low fraction with low HBM and FP64 fractions is the signature of the binding limit: the
    SM's instruction delivery to 16 distinct straight-line warp streams (~0.5-0.75
    warp-instructions per cycle per busy SM, measured per phase in profiles/r2_phase_trace/).
    """
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            d = json.load(fh).get(workload)
    except (OSError, ValueError):
        return None
    if not d or d.get("batch") != B or not d.get("warp_instr_per_step"):
        return None
    mhz = (clocks or {}).get("sm_max_mhz") or 1965.0
    peak = 148 * 4 * mhz * 1e6
    achieved = d["warp_instr_per_step"] / mean_s
    busy_sms = min(148, -(-B // 32))
    return {"achieved": achieved, "peak": peak, "unit": "warp-instr/s", "frac": achieved / peak,
            "ipc_per_busy_sm": achieved / (busy_sms * mhz * 1e6), "busy_sms": busy_sms,
            "warp_instr_per_step": d["warp_instr_per_step"], "source": d["source"].split(":")[0]}


def committed_traffic(workload, info, B):
    """DRAM bytes per step from the committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            d = json.load(fh).get(workload)
        if d and d.get("batch", 4096) == B:
            return d["dram_bytes_per_eval"] * B, d["source"]
    except (OSError, ValueError, KeyError):
        pass
    return None, None


PIPE_DEPTH = 3
SECONDARY = (("cartpole_rk4", 1_000_000), ("pendulum", 1_000_000), ("humanoid_rbd", 65536), ("srbm_mpc", 65536))


def secondary_points(dev, local, hbm_gbs, steps=5):
    """Other BASELINE configs at scale, device-resident, L2 flushed per step
    (small tapes are the HBM-bound ones the metric's "% HBM roofline" is about)."""
    import torch

    import oracle
    import paper_2408_09662_b200 as vsb
    import workloads

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    out = []
    for name, B in SECONDARY:
        tape = workloads.load_tape(name)
        plan = vsb.get_plan(tape)
        ins = workloads.make_inputs(name, B, seed=2000)
        nin, nout = tape.nnz_in, tape.nnz_out
        in_off = np.concatenate([[0], np.cumsum(np.asarray(nin, dtype=np.int64) * B)])
        out_off = np.concatenate([[0], np.cumsum(np.asarray(nout, dtype=np.int64) * B)])
        d_in = torch.tensor(np.concatenate([v.ravel() for v in ins]), device=dev)
        d_out = torch.empty(int(out_off[-1]), dtype=torch.float64, device=dev)

        def step():
            plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, 0, B, local, stream.cuda_stream)

        for _ in range(3):
            flush.zero_()
            step()
        ms = []
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        t = statistics.median(ms) / 1e3
        rows = np.random.default_rng(0).choice(B, size=16, replace=False)
        ref = oracle.batch_eval(tape, [v[rows] for v in ins])
        got = d_out.cpu().numpy()
        worst = 0.0
        for j in range(tape.n_out):
            g = got[out_off[j]:out_off[j + 1]].reshape(B, nout[j])[rows]
            worst = max(worst, float(np.nanmax(np.abs(g - ref[j]) / np.maximum(np.abs(ref[j]), 1.0))))
        info = plan.info
        gbs = 8 * (sum(nin) + sum(nout)) * B / t / 1e9
        out.append({"workload": name, "batch": B, "value": B / t, "unit": "evals/s", "ms_per_step": t * 1e3,
                    "hbm_gbs": gbs, "hbm_frac": gbs / hbm_gbs, "team": info["team"], "n_chunks": info["n_chunks"],
                    "max_rel_err_16_rows": worst})
        del d_in, d_out
    out.append(rollout_point(dev))
    return out


def rollout_point(dev, B=10000, K=100, reps=5):
    """quadsim.rollout_batch's closed loop (quad_step, one broadcast
    theta) as one device-resident rollout -- hoisted pre tape + fused K-step kernel."""
    import torch

    import workloads
    from paper_2408_09662_b200.rollout import Rollout

    tape = workloads.load_tape("quad_step")
    ins = workloads.make_inputs("quad_step", B, seed=2001)
    theta = np.repeat(ins[1][:1], B, axis=0)
    r = Rollout(tape, B, K, device=dev)
    r.set(torch.tensor(ins[0], device=dev), [torch.tensor(theta, device=dev)])
    r.run()
    torch.cuda.synchronize(dev)
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r.run()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    t = statistics.median(ms) / 1e3
    return {"workload": "quad_step rollout (quadsim.rollout_batch, one theta)", "batch": B, "steps": K,
            "value": B * K / t, "unit": "env-steps/s", "ms_per_rollout": t * 1e3,
            "hoisted_rows": r.split.hoisted_rows if r.split is not None else 0, "fused": r.fused,
            "launches_per_rollout": r.launches_per_run}


def batch_sweep(dev, local, hbm_gbs, steps=5):
    """BASELINE metric's batch axis: evals/s of the headline tape and of the small
    HBM-bound tape at B = 1e2 ... 1e6 (device-resident, L2 flushed per step)."""
    import torch

    import paper_2408_09662_b200 as vsb
    import workloads

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    rows = []
    for name, batches in (("srbm_mpc", (100, 1000, 4096, 10_000, 65_536, 100_000, 1_000_000)),
                          ("cartpole_rk4", (100, 1000, 4096, 10_000, 65_536, 100_000, 1_000_000))):
        tape = workloads.load_tape(name)
        plan = vsb.get_plan(tape)
        nin, nout = tape.nnz_in, tape.nnz_out
        for B in batches:
            ins = workloads.make_inputs(name, B, seed=4000)
            in_off = np.concatenate([[0], np.cumsum(np.asarray(nin, dtype=np.int64) * B)])
            out_off = np.concatenate([[0], np.cumsum(np.asarray(nout, dtype=np.int64) * B)])
            d_in = torch.tensor(np.concatenate([v.ravel() for v in ins]), device=dev)
            d_out = torch.empty(int(out_off[-1]), dtype=torch.float64, device=dev)

            def step():
                plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, 0, B, local, stream.cuda_stream)

            ms = []
            for k in range(3 + steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                step()
                b.record(stream)
                b.synchronize()
                if k >= 3:
                    ms.append(a.elapsed_time(b))
            t = statistics.median(ms) / 1e3
            gbs = 8 * (sum(nin) + sum(nout)) * B / t / 1e9
            rows.append({"workload": name, "batch": B, "value": B / t, "unit": "evals/s", "ms_per_step": t * 1e3,
                         "hbm_frac": gbs / hbm_gbs})
            del d_in, d_out
    return rows


def parity_all_rows(tape, inputs, got_flat, out_off, B):
    """Every row of the timed batch against the CPU oracle (fp64 contract 1e-12 relative)."""
    import oracle

    ref = oracle.batch_eval(tape, inputs, n_threads=len(os.sched_getaffinity(0)))
    worst, bad = 0.0, 0
    for j, nz in enumerate(tape.nnz_out):
        g = got_flat[out_off[j]:out_off[j + 1]].reshape(B, nz)
        with np.errstate(invalid="ignore"):
            err = np.abs(g - ref[j]) / np.maximum(np.abs(ref[j]), 1.0)
        err[np.isnan(g) & np.isnan(ref[j])] = 0.0
        if err.size:
            worst = max(worst, float(np.nanmax(err)))
            bad += int(np.count_nonzero(~(err <= 1e-12)))
    bits = all(np.array_equal(got_flat[out_off[j]:out_off[j + 1]].reshape(B, nz).view(np.uint64),
                              ref[j].view(np.uint64)) for j, nz in enumerate(tape.nnz_out))
    return {"rows_checked": int(B), "max_rel_err": worst, "violations": bad, "bitwise_identical": bool(bits),
            "tolerance": 1e-12, "ok": bad == 0}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2408_09662_b200 as vsb
    import workloads
    from paper_2408_09662_b200.dist import batch_eval_ranks, max_over_ranks, shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    tape = workloads.load_tape(args.workload)
    if args.global_batch:
        # strong scaling (config 4): one global batch split B*k//W over ranks
        lo, hi = shard_bounds(args.global_batch, world, rank)
        B = hi - lo
        total_instances = args.global_batch
    else:
        B = args.batch
        total_instances = world * B
    inputs = workloads.make_inputs(args.workload, B, seed=1000 + rank)
    opts = {}
    for k in ("block", "chunk_ops", "team", "min_blocks", "groups", "cluster", "outline", "phase_cost"):
        if getattr(args, k):
            opts[k] = getattr(args, k)
    plan = vsb.get_plan(tape, **opts)
    info = plan.info

    nin, nout = tape.nnz_in, tape.nnz_out
    in_off = np.concatenate([[0], np.cumsum(np.asarray(nin, dtype=np.int64) * B)])
    out_off = np.concatenate([[0], np.cumsum(np.asarray(nout, dtype=np.int64) * B)])
    d_in = torch.tensor(np.concatenate([v.ravel() for v in inputs]) if nin else np.zeros(1), device=dev)
    d_out = torch.empty(max(1, int(out_off[-1])), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, 0, B, local, sptr)

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for s, e in evs:
        flush.zero_()
        s.record(stream)
        step()
        e.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = max_over_ranks(sum(s.elapsed_time(e) for s, e in evs), device=dev)
    clocks = sampler.stop() if sampler else None

    # parity of the timed configuration: every row of this rank's batch vs the CPU oracle
    parity = parity_all_rows(tape, inputs, d_out.cpu().numpy(), out_off, B) if rank == 0 else None

    # end to end through the reference-shaped public API (pinned host buffers); strong
    # scaling runs dist.batch_eval_ranks over one global workspace (shard, final gather)
    if args.global_batch:
        e2e_tape_ws = vsb.BatchWorkspace(tape, args.global_batch)
        g_in = workloads.make_inputs(args.workload, args.global_batch, seed=1000) if world > 1 else inputs
        for i, v in enumerate(g_in):
            e2e_tape_ws.set_input(i, v)

        def e2e_call():
            batch_eval_ranks(tape, e2e_tape_ws, device=local, plan_options=opts or None)
    else:
        e2e_tape_ws = vsb.BatchWorkspace(tape, B)
        for i, v in enumerate(inputs):
            e2e_tape_ws.set_input(i, v)

        def e2e_call():
            vsb.batch_eval(tape, e2e_tape_ws, device=local, plan_options=opts or None)
    # warm-up >= 1 s: the PCIe link of an idle B200 needs ~0.5 s of traffic before pinned H2D
    # reaches full speed (tools/h2d_probe2.py: 15-30 GB/s cold, 54 GB/s warm)
    t_warm = time.perf_counter()
    while time.perf_counter() - t_warm < 1.0:
        e2e_call()
    if world > 1:
        dist.barrier()
    e2e_steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_sync_s = max_over_ranks(time.perf_counter() - t0, device=dev)
    if world > 1:
        dist.barrier()

    # the same steps as a stream of batches through BatchPipeline (vsb_pipe_*): every step
    # still copies its inputs from pinned host memory and its outputs back, but step k+1's
    # H2D and step k-1's D2H overlap step k's kernels.  PIPE_DEPTH workspaces rotate (a
    # step's host buffers are reused only after its ticket was waited for); depth 3 reaches
    # the device rate on srbm_mpc B=4096, depth 2 95% of it (profiles/r2_27_pipe.jsonl)
    pipe_steps = max(3, min(args.steps, 50))
    pipe_ws = None
    if not args.global_batch:
        pipe_ws = [e2e_tape_ws] + [vsb.BatchWorkspace(tape, B) for _ in range(PIPE_DEPTH - 1)]
        for w in pipe_ws[1:]:
            for i, v in enumerate(inputs):
                w.set_input(i, v)
        pipe = vsb.BatchPipeline(tape, depth=PIPE_DEPTH, device=local, plan_options=opts or None)

        def pipe_run(k_steps):
            tickets = []
            for k in range(k_steps):
                if k >= PIPE_DEPTH:
                    pipe.wait(tickets[k - PIPE_DEPTH])
                tickets.append(pipe.submit(pipe_ws[k % PIPE_DEPTH]))
            for t in tickets[max(0, k_steps - PIPE_DEPTH):]:
                pipe.wait(t)

        t_warm = time.perf_counter()
        while time.perf_counter() - t_warm < 0.5:
            pipe_run(4)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        pipe_run(pipe_steps)
        e2e_pipe_s = max_over_ranks(time.perf_counter() - t0, device=dev)
        pipe.close()
        if world > 1:
            dist.barrier()
        # the pipelined outputs are the device run's bits
        dev_out = d_out.cpu().numpy()
        pipe_match = bool(all(np.array_equal(w._out_buf.view(np.uint64), dev_out[: w._out_buf.size].view(np.uint64))
                              for w in pipe_ws)) if dev_out.size >= pipe_ws[0]._out_buf.size else None

    if rank != 0:
        dist.destroy_process_group()
        return

    hbm_gbs, sm_max_mhz, peak_kind = load_peaks()
    bytes_eval = 8 * (sum(nin) + sum(nout))
    mean_s = total_ms / 1e3 / args.steps
    achieved_gbs = bytes_eval * B / mean_s / 1e9
    ops_eval = info["n_arith_rows"]
    fp64_peak = 148 * 64 * sm_max_mhz * 1e6 / 1e12  # one non-fused DP op per lane per clock
    fp64_achieved = ops_eval * B / mean_s / 1e12
    value = total_instances * args.steps / (total_ms / 1e3)
    e2e_sync_value = total_instances * e2e_steps / e2e_sync_s
    if pipe_ws is not None:
        e2e_value = total_instances * pipe_steps / e2e_pipe_s
        e2e_api = (f"paper_2408_09662_b200.BatchPipeline(tape, depth={PIPE_DEPTH}).submit(BatchWorkspace)"
                   " [pinned host buffers]")
        e2e_timing = (f"{pipe_steps} pipelined steps ({PIPE_DEPTH} workspaces, {PIPE_DEPTH} in flight), host wall clock"
                      " from the first submit to the last wait, max over ranks")
    else:
        e2e_value = e2e_sync_value
        e2e_api = "paper_2408_09662_b200.dist.batch_eval_ranks(tape, BatchWorkspace) [pinned host buffers]"
        e2e_timing = f"{e2e_steps} synchronous calls, host wall clock, max over ranks"

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        Bs = cpu_sample_batch(tape, B, threads)
        rate, reps, secs = cpu_baseline(tape, [v[:Bs] for v in inputs], args.cpu_seconds, threads)
        Bs1 = cpu_sample_batch(tape, B, 1)
        rate1, _, _ = cpu_baseline(tape, [v[:Bs1] for v in inputs], 2.0, 1)
        cpu = {"value": rate, "unit": "evals/s", "cores": threads, "kind": "port",
               "sample": f"{Bs} instances x {reps} calls ({secs:.1f} s), W={threads} pthreads, "
                         "oracle/vs_oracle.c restating vecsym run_range/batch_eval",
               "w1_value": rate1, "speedup_value_vs_cpu": value / rate, "speedup_e2e_vs_cpu": e2e_value / rate,
               "reference_numba": None if args.no_numba else reference_numba(tape, inputs, threads)}

    issue = issue_roof(args.workload, B, mean_s, clocks) if info.get("team") else None
    secondary = sweep = None
    if world == 1 and not args.no_secondary:
        secondary = secondary_points(dev, local, hbm_gbs)
        sweep = batch_sweep(dev, local, hbm_gbs)
    traffic, traffic_src = committed_traffic(args.workload, info, B)

    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.global_batch else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": arm_config(args, world, tape),
        "workload_detail": {"arith_ops_per_eval": ops_eval, "io_bytes_per_eval": bytes_eval,
                            "l2": "flushed (256 MiB write) before every timed step, outside the events",
                            "plan": {k: info[k] for k in ("team", "n_chunks", "block", "scratch_slots", "scratch_loads",
                                                          "scratch_stores", "max_regs", "max_local_bytes",
                                                          "phases", "est_efficiency", "code_bytes")}},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_gbs, "unit": "GB/s",
                     "frac": achieved_gbs / hbm_gbs, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind,
                     "note": "achieved = algorithmic I/O bytes 8*(sum nnz_in + sum nnz_out) per eval x batch over"
                             " the whole kernel chain of one step (CUDA events); traffic = ncu dram bytes of the same"
                             " chain per step. Neither HBM nor the FP64 pipe binds a large tape at this batch: the"
                             " binding limit is instruction delivery to 16 distinct straight-line warp streams per SM"
                             " (issue, DESIGN.md 4.4c)",
                     "issue": issue,
                     "fp64": {"achieved": fp64_achieved, "peak": fp64_peak, "unit": "Tops/s",
                              "frac": fp64_achieved / fp64_peak,
                              "peak_def": "148 SM x 64 FP64 lanes x sm_max_mhz, 1 op/lane/clk (no FMA: --fmad=false)"}},
        "e2e": {"value": e2e_value, "unit": "evals/s",
                "h2d_bytes_per_step": 8 * sum(nin) * total_instances, "d2h_bytes_per_step": 8 * sum(nout) * total_instances,
                "api": e2e_api, "timing": e2e_timing,
                "sync": {"value": e2e_sync_value, "unit": "evals/s",
                         "api": "paper_2408_09662_b200.batch_eval(tape, BatchWorkspace) [pinned host buffers]"
                                if not args.global_batch else e2e_api,
                         "timing": f"{e2e_steps} synchronous calls (copy, kernels, copy back; one call at a time)"},
                "outputs_match_device_run": pipe_match if pipe_ws is not None else None},
        "gpu_launches": args.steps * plan.launches_per_eval(B),
        "clocks": clocks,
        "parity": parity,
        "cpu_baseline": cpu,
        "secondary": secondary,
        "batch_sweep": sweep,
    }
    if world > 1:
        dist.destroy_process_group()   # before printing: NCCL's INFO lines must not follow the JSON line
    print(json.dumps(line), flush=True)


def run_inprocess(args):
    """One process driving N GPUs through the in-process sharder (``batch_eval(devices=...)``,
    ``vsb_eval_host_sharded``: contiguous shards, a host thread + streams per GPU)."""
    import torch

    import paper_2408_09662_b200 as vsb
    import workloads

    n = min(args.gpus, torch.cuda.device_count())
    tape = workloads.load_tape(args.workload)
    total = args.global_batch or args.batch * n
    ws = vsb.BatchWorkspace(tape, total)
    for i, v in enumerate(workloads.make_inputs(args.workload, total, seed=1000)):
        ws.set_input(i, v)
    devs = list(range(n))
    t_warm = time.perf_counter()
    while time.perf_counter() - t_warm < 1.0:
        vsb.batch_eval(tape, ws, devices=devs)
    steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(steps):
        vsb.batch_eval(tape, ws, devices=devs)
    dt = time.perf_counter() - t0
    nin, nout = tape.nnz_in, tape.nnz_out
    print(json.dumps({"metric": METRIC, "value": total * steps / dt, "unit": "evals/s", "n_gpus": n,
                      "steps": steps, "warmup": 1, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
                      "scaling": "strong" if args.global_batch else "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": arm_config(args, n, tape),
                      "e2e": {"value": total * steps / dt, "unit": "evals/s", "h2d_bytes_per_step": 8 * sum(nin) * total,
                              "d2h_bytes_per_step": 8 * sum(nout) * total,
                              "api": f"paper_2408_09662_b200.batch_eval(tape, BatchWorkspace, devices={devs})"}}),
          flush=True)


def spawn_ranks(args):
    """`--gpus N` outside torchrun: re-launch this script with one process per GPU."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # NCCL's init lines name the rank count
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="srbm_mpc")
    ap.add_argument("--batch", type=int, default=4096, help="instances per GPU (weak scaling)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="total instances split over the GPUs (strong scaling, config 4)")
    ap.add_argument("--team", type=int, default=0, help="warps per 32-instance team (0 = auto)")
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--chunk-ops", type=int, default=0)
    ap.add_argument("--min-blocks", type=int, default=0)
    ap.add_argument("--groups", type=int, default=0, help="team mode: 32-instance groups per CTA")
    ap.add_argument("--cluster", type=int, default=0, help="team mode: CTAs per thread-block cluster")
    ap.add_argument("--outline", type=int, default=0, help="outlined DIV/trig subroutines (0 auto, -1 none)")
    ap.add_argument("--phase-cost", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-w1", action="store_true", help="also time the oracle with one thread")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the other-config points (cartpole/pendulum 1e6, humanoid/srbm 65536)")
    ap.add_argument("--no-numba", action="store_true", help="skip timing the reference's numba evaluator")
    ap.add_argument("--inprocess", action="store_true",
                    help="N GPUs from one process via batch_eval(devices=range(N)) (e2e only)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.inprocess:
        run_inprocess(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    else:
        if int(os.environ.get("WORLD_SIZE", "1")) > 1:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        run_ours(args)


if __name__ == "__main__":
    main()
