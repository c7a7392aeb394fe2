"""Reference-compatible batched runtime on B200.

Same operator surface as ``vecsym.batchrt`` (/root/reference/pkg/src/vecsym/
batchrt.py:25-30): ``BatchWorkspace``, ``batch_eval``, ``serial_eval``,
``default_thread_count``, with the same buffer layout, argument meaning and
error messages, so callers (quadsim rollouts, the bench harness, the CLI)
switch by changing the import.  Evaluation runs on the GPU through the
C ABI (``vsb_eval_host``: pinned H2D -> sm_100a kernel chain -> D2H,
pipelined); there is no CPU fallback -- a missing extension or device
raises.

Differences, all additive: ``device=`` / ``devices=`` select GPUs (the
latter shards the batch with the reference's contiguous-chunk rule,
batchrt.py:189-191); ``n_threads`` is validated exactly as the reference
does but does not change the GPU execution; host buffers are pinned.
"""

from __future__ import annotations

import ctypes
import os
import weakref

import numpy as np

from . import _native
from .plan import get_plan
from .tape import InstructionTape, as_tape

__all__ = ["BatchWorkspace", "serial_eval", "batch_eval", "default_thread_count", "BatchPipeline"]


def default_thread_count() -> int:
    """Mirror of batchrt.default_thread_count (batchrt.py:33-50): the
    ``VECSYM_THREADS`` override is honoured and validated identically."""
    env = os.environ.get("VECSYM_THREADS")
    if env is not None and env.strip():
        try:
            n = int(env)
        except ValueError:
            raise ValueError(f"VECSYM_THREADS must be a positive integer, got {env!r}") from None
        if n < 1:
            raise ValueError(f"VECSYM_THREADS must be a positive integer, got {env!r}")
        return n
    return os.cpu_count() or 1


def _offsets(nnz, batch_size: int) -> np.ndarray:
    off = np.zeros(len(nnz) + 1, dtype=np.int64)
    np.cumsum(np.asarray(nnz, dtype=np.int64) * batch_size, out=off[1:])
    return off


def _pinned_zeros(n: int, dtype) -> np.ndarray:
    """Zero-filled page-locked host array (cudaHostAlloc via the C ABI) so
    host<->device copies are asynchronous DMA; plain memory without a driver."""
    itemsize = np.dtype(dtype).itemsize
    nbytes = max(1, n) * itemsize
    L = _native.lib()
    ptr = ctypes.c_void_p()
    if L.vsb_host_alloc(ctypes.byref(ptr), nbytes) != _native.VSB_OK or not ptr.value:
        return np.zeros(n, dtype=dtype)
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dtype, count=max(1, n))[:n]
    arr[:] = 0
    weakref.finalize(buf, L.vsb_host_free, ctypes.c_void_p(ptr.value))
    return arr


class BatchWorkspace:
    """Preallocated env-major buffers for one (tape, batch size) pairing
    (batchrt.py:78-169).  ``inputs[i]`` / ``outputs[j]`` are flat views of
    length ``batch_size * nnz`` with element e's k-th nonzero at
    ``e * nnz + k``.  ``work`` exists for API compatibility only (the GPU keeps
    the work vector in registers) and is allocated on first access."""

    __slots__ = ("batch_size", "inputs", "outputs", "dtype", "_in_buf", "_out_buf", "_in_off", "_out_off",
                 "_nnz_in", "_nnz_out", "_n_w", "_tape_name", "_work", "__weakref__")

    def __init__(self, tape, batch_size: int, dtype=np.float64):
        tape = as_tape(tape)
        batch_size = int(batch_size)
        if batch_size < 1:
            raise ValueError(f"batch_size must be >= 1, got {batch_size}")
        self.batch_size = batch_size
        self.dtype = np.dtype(dtype)
        self._n_w = tape.n_w
        self._nnz_in = tuple(tape.nnz_in)
        self._nnz_out = tuple(tape.nnz_out)
        self._tape_name = tape.name
        self._in_off = _offsets(self._nnz_in, batch_size)
        self._out_off = _offsets(self._nnz_out, batch_size)
        self._in_buf = _pinned_zeros(int(self._in_off[-1]), self.dtype)
        self._out_buf = _pinned_zeros(int(self._out_off[-1]), self.dtype)
        self._work = None
        self.inputs = [self._in_buf[int(self._in_off[i]) : int(self._in_off[i + 1])] for i in range(len(self._nnz_in))]
        self.outputs = [self._out_buf[int(self._out_off[j]) : int(self._out_off[j + 1])] for j in range(len(self._nnz_out))]

    @property
    def work(self) -> np.ndarray:
        if self._work is None:
            self._work = np.zeros(self.batch_size * self._n_w, dtype=self.dtype)
        return self._work

    def input_matrix(self, i: int) -> np.ndarray:
        """Writable (batch_size, nnz_in[i]) view of input ``i``."""
        return self.inputs[i].reshape(self.batch_size, self._nnz_in[i])

    def output_matrix(self, j: int) -> np.ndarray:
        """(batch_size, nnz_out[j]) view of output ``j``."""
        return self.outputs[j].reshape(self.batch_size, self._nnz_out[j])

    def set_input(self, i: int, values) -> None:
        """One instance's nonzeros (broadcast) or a (batch_size, nnz) array."""
        v = np.asarray(values, dtype=self.dtype)
        nnz = self._nnz_in[i]
        if v.ndim <= 1:
            if v.size != nnz:
                raise ValueError(f"input {i}: expected {nnz} values, got {v.size}")
            self.input_matrix(i)[:, :] = v.ravel()
        else:
            if v.shape != (self.batch_size, nnz):
                raise ValueError(f"input {i}: expected shape ({self.batch_size}, {nnz}), got {v.shape}")
            self.input_matrix(i)[:, :] = v

    def matches(self, tape) -> bool:
        return (self._n_w == tape.n_w and self._nnz_in == tuple(tape.nnz_in)
                and self._nnz_out == tuple(tape.nnz_out))

    def __repr__(self) -> str:
        return (f"BatchWorkspace(batch_size={self.batch_size}, n_w={self._n_w}, "
                f"nnz_in={list(self._nnz_in)}, nnz_out={list(self._nnz_out)})")


def _plan_for(tape, ws: BatchWorkspace, plan_options):
    dtype = "float32" if ws.dtype == np.float32 else "float64"
    return get_plan(tape, dtype=dtype, **(plan_options or {}))


def batch_eval(tape, ws: BatchWorkspace, n_threads: int | None = None, *, device: int = 0,
               devices=None, plan_options: dict | None = None) -> list[np.ndarray]:
    """Evaluate every element of ``ws`` through ``tape`` on the GPU (batchrt.py:194-244).

    Writes ``ws.outputs`` in place and returns them.  ``devices`` (a list of
    CUDA ordinals) shards the batch across GPUs with no collective.
    """
    tape = as_tape(tape)
    if not ws.matches(tape):
        raise ValueError(
            f"workspace/tape mismatch: workspace is laid out for n_w={ws._n_w}, "
            f"nnz_in={list(ws._nnz_in)}, nnz_out={list(ws._nnz_out)} but tape "
            f"{tape.name!r} needs n_w={tape.n_w}, nnz_in={tape.nnz_in}, nnz_out={tape.nnz_out}"
        )
    if n_threads is not None and n_threads < 1:
        raise ValueError(f"n_threads must be >= 1, got {n_threads}")
    plan = _plan_for(tape, ws, plan_options)
    in_ptr = ws._in_buf.ctypes.data
    out_ptr = ws._out_buf.ctypes.data
    if devices is not None and len(devices) > 1:
        plan.eval_host_sharded(in_ptr, ws._in_off, out_ptr, ws._out_off, 0, ws.batch_size, list(devices))
    else:
        dev = int(devices[0]) if devices else int(device)
        plan.eval_host(in_ptr, ws._in_off, out_ptr, ws._out_off, 0, ws.batch_size, dev)
    return ws.outputs


class BatchPipeline:
    """Asynchronous ``batch_eval`` over a stream of workspaces (``vsb_pipe_*``).

    ``submit(ws)`` enqueues one batch -- pinned H2D, the kernel chain, D2H -- and
    returns a ticket without waiting; ``wait(ticket)`` / ``drain()`` block until the
    outputs are in ``ws.outputs``.  With ``depth`` batches in flight the next batch's
    input copy and the previous batch's output copy overlap the current batch's
    kernels, so a stream of batches costs max(H2D, kernels, D2H) per batch instead of
    their sum.  A submitted workspace must not be modified or read until its ticket is
    waited for.  Additive to the reference, whose ``batch_eval`` (batchrt.py:194-244)
    is synchronous; results are the same bits as ``batch_eval``.
    """

    def __init__(self, tape, *, depth: int = 2, device: int = 0, plan_options: dict | None = None):
        self.tape = as_tape(tape)
        if not 1 <= int(depth) <= 16:
            raise ValueError(f"depth must be in [1, 16], got {depth}")
        self.device = int(device)
        self._plan_options = plan_options
        self._plan = None
        self._h = None
        self._depth = int(depth)
        self._pending: dict[int, BatchWorkspace] = {}

    def _open(self, ws: BatchWorkspace) -> None:
        if self._h is not None:
            return
        self._plan = _plan_for(self.tape, ws, self._plan_options)
        h = ctypes.c_void_p()
        _native.check(_native.lib().vsb_pipe_create(self._plan.handle, self.device, self._depth, ctypes.byref(h)))
        self._h = h
        self._finalizer = weakref.finalize(self, _native.lib().vsb_pipe_destroy, h)

    def submit(self, ws: BatchWorkspace) -> int:
        if not ws.matches(self.tape):
            raise ValueError(
                f"workspace/tape mismatch: workspace is laid out for n_w={ws._n_w}, "
                f"nnz_in={list(ws._nnz_in)}, nnz_out={list(ws._nnz_out)} but tape "
                f"{self.tape.name!r} needs n_w={self.tape.n_w}, nnz_in={self.tape.nnz_in}, nnz_out={self.tape.nnz_out}"
            )
        self._open(ws)
        ticket = ctypes.c_int64(-1)
        i64p = ctypes.POINTER(ctypes.c_int64)
        _native.check(_native.lib().vsb_pipe_submit(
            self._h, ctypes.c_void_p(ws._in_buf.ctypes.data), ws._in_off.ctypes.data_as(i64p),
            ctypes.c_void_p(ws._out_buf.ctypes.data), ws._out_off.ctypes.data_as(i64p),
            0, ws.batch_size, ctypes.byref(ticket)))
        self._pending[ticket.value] = ws   # keeps the host buffers alive while in flight
        return ticket.value

    def wait(self, ticket: int) -> list[np.ndarray]:
        if ticket not in self._pending:
            raise ValueError(f"unknown or already waited ticket {ticket}")
        _native.check(_native.lib().vsb_pipe_wait(self._h, int(ticket)))
        return self._pending.pop(ticket).outputs

    def drain(self) -> None:
        if self._h is not None:
            _native.check(_native.lib().vsb_pipe_drain(self._h))
        self._pending.clear()

    def close(self) -> None:
        if self._h is not None:
            self._finalizer()
            self._h = None
        self._pending.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.drain()
        self.close()


def serial_eval(tape, input_values, *, device: int = 0) -> list[np.ndarray]:
    """One instance (batchrt.py:172-186), evaluated by the same GPU kernels."""
    tape = as_tape(tape)
    ins = [np.ascontiguousarray(v, dtype=np.float64).ravel() for v in input_values]
    if len(ins) != tape.n_in:
        raise ValueError(f"expected {tape.n_in} inputs, got {len(ins)}")
    for k, (v, nz) in enumerate(zip(ins, tape.nnz_in)):
        if v.size != nz:
            raise ValueError(f"input {k}: expected {nz} values, got {v.size}")
    ws = BatchWorkspace(tape, 1)
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    batch_eval(tape, ws, device=device)
    return [o.copy() for o in ws.outputs]
