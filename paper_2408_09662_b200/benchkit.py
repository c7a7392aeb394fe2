"""Serial-vs-batched timing harness on the B200 path (the reference's
``vecsym.bench`` methodology, /root/reference/pkg/src/vecsym/bench.py:133-225).

Same protocol: two warm-up calls, median of >= 5 repetitions, every sample
looped until it spans >= 100 timer ticks (``_median_call_time``,
bench.py:133-156); ``t_serial_total`` = batch x the median single-instance
``serial_eval`` time, ``t_batch`` = the median ``batch_eval`` time, and
``speedup`` is their quotient, never measured independently (bench.py:1-9).
Here both columns run on the GPU through pinned host buffers, so they include
the host<->device copies; ``t_device`` (optional column) is the kernel chain
alone on device-resident data (CUDA events).  The reference's graded
``gen_ldlt_case`` builder is an offline symbolic producer (out of scope); cases
are saved tapes.
"""

from __future__ import annotations

import csv
import statistics
import time
from typing import NamedTuple

import numpy as np

from .batchrt import BatchWorkspace, batch_eval, serial_eval
from .tape import as_tape

__all__ = ["BenchRecord", "MIN_REPETITIONS", "WARMUP_CALLS", "CSV_HEADER", "run_benchmark", "write_bench_csv"]

MIN_REPETITIONS = 5
WARMUP_CALLS = 2
_MIN_TIMER_TICKS = 100
_MAX_INNER_CALLS = 1_000_000_000
CSV_HEADER = ("n_instructions", "batch_size", "n_threads", "t_serial_total", "t_batch", "speedup")


class BenchRecord(NamedTuple):
    """One (case, batch) row of bench.csv: the reference's six columns (``speedup``
    derived, bench.py:1-9) plus ``repetitions`` and the optional device-only time."""

    n_instructions: int
    batch_size: int
    n_threads: int
    t_serial_total: float
    t_batch: float
    repetitions: int
    t_device: float | None = None

    @property
    def speedup(self) -> float:
        return self.t_serial_total / self.t_batch


def _record(*fields, **kw) -> BenchRecord:
    rec = BenchRecord(*fields, **kw)
    if rec.t_serial_total <= 0 or rec.t_batch <= 0:
        raise ValueError("timings must be positive")
    return rec


def _median_call_time(fn, repetitions: int) -> float:
    """Median seconds per call over ``repetitions`` samples; each sample runs the call
    enough times (a power of ten) to span >= 100 ticks of the host timer."""
    need = time.get_clock_info("perf_counter").resolution * _MIN_TIMER_TICKS

    def sample(calls: int) -> float:
        t0 = time.perf_counter()
        for _ in range(calls):
            fn()
        return time.perf_counter() - t0

    calls, first = 1, sample(1)
    while first < need:
        if calls >= _MAX_INNER_CALLS:
            raise RuntimeError(f"timer resolution insufficient: {calls} calls span {first:.3e}s < {need:.3e}s")
        calls *= 10
        first = sample(calls)
    return statistics.median([first / calls] + [sample(calls) / calls for _ in range(repetitions - 1)])


def _device_time(tape, ws: BatchWorkspace, repetitions: int, device: int) -> float:
    """Kernel chain alone on device-resident copies of the workspace (CUDA events)."""
    import torch

    from .plan import get_plan

    plan = get_plan(tape, dtype="float32" if ws.dtype == np.float32 else "float64")
    dev = torch.device("cuda", device)
    d_in = torch.from_numpy(np.asarray(ws._in_buf)).to(dev) if ws._in_buf.size else torch.zeros(1, device=dev)
    d_out = torch.empty(max(1, ws._out_buf.size), dtype=d_in.dtype, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.eval_device(d_in.data_ptr(), ws._in_off, d_out.data_ptr(), ws._out_off, 0, ws.batch_size, device,
                         stream.cuda_stream)

    for _ in range(WARMUP_CALLS):
        step()
    ms = []
    for _ in range(repetitions):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ms)


def run_benchmark(cases, batch_sizes, n_threads: int | None = None, repetitions: int = MIN_REPETITIONS,
                  rng_seed: int = 0, device: int = 0, device_column: bool = False) -> list[BenchRecord]:
    """Time every (case, batch size) pair (bench.py:159-210).

    ``cases``: iterable of ``(tape, inputs)`` with ``inputs`` one instance's
    nonzeros per input (broadcast over the batch like the reference's
    ``np.tile``), or bare tapes (random N(0,1) inputs from ``rng_seed``).
    """
    cases = list(cases)
    batch_sizes = [int(b) for b in batch_sizes]
    if not cases or not batch_sizes:
        raise ValueError("need at least one case and one batch size")
    if any(b < 1 for b in batch_sizes):
        raise ValueError("batch sizes must be >= 1")
    if repetitions < MIN_REPETITIONS:
        raise ValueError(f"repetitions must be >= {MIN_REPETITIONS}, got {repetitions}")
    n_threads = 1 if n_threads is None else int(n_threads)   # host threads play no part on the GPU path
    rng = np.random.default_rng(rng_seed)
    records = []
    for case in cases:
        tape, inputs = case if isinstance(case, tuple) else (case, None)
        tape = as_tape(tape)
        if inputs is None:
            inputs = [rng.normal(size=nz) for nz in tape.nnz_in]
        for _ in range(WARMUP_CALLS):
            serial_eval(tape, inputs, device=device)
        t_serial = _median_call_time(lambda: serial_eval(tape, inputs, device=device), repetitions)
        for batch in batch_sizes:
            ws = BatchWorkspace(tape, batch)
            for i, v in enumerate(inputs):
                ws.set_input(i, np.tile(np.asarray(v, dtype=float).ravel(), (batch, 1)))
            for _ in range(WARMUP_CALLS):
                batch_eval(tape, ws, n_threads=n_threads, device=device)
            t_batch = _median_call_time(lambda: batch_eval(tape, ws, n_threads=n_threads, device=device), repetitions)
            t_dev = _device_time(tape, ws, repetitions, device) if device_column else None
            records.append(_record(tape.n_arith, batch, n_threads, batch * t_serial, t_batch, repetitions, t_dev))
    return records


def write_bench_csv(path, records, device_column: bool = False) -> None:
    """The reference's fixed six-column header (bench.py:213-225), plus ``t_device`` on request."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(CSV_HEADER + (("t_device",) if device_column else ()))
        for rec in records:
            row = [rec.n_instructions, rec.batch_size, rec.n_threads, repr(rec.t_serial_total), repr(rec.t_batch),
                   repr(rec.speedup)]
            if device_column:
                row.append(repr(rec.t_device))
            writer.writerow(row)
