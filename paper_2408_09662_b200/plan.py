"""Compiled evaluation plans (a thin owner of a native ``vsb_plan``).

A plan is the B200 replacement for the reference's per-call tape walk
(``_kernels.run_range``, _kernels.py:54-206): the tape is SSA-renamed,
cut into chained kernels when large, emitted as sm_100a CUDA and compiled
once by NVRTC (cached on disk by content hash).  Plans are cached per
(tape digest, options) so the reference-shaped ``batch_eval`` API never
recompiles.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native
from ._native import Options, PlanInfo, check
from .tape import InstructionTape, as_tape

__all__ = ["Plan", "get_plan", "clear_plan_cache"]

_DTYPES = {"float64": _native.VSB_F64, "f64": _native.VSB_F64, "float32": _native.VSB_F32, "f32": _native.VSB_F32}


def _dtype_code(dtype) -> int:
    key = str(dtype).replace("torch.", "").replace("numpy.", "")
    if key not in _DTYPES:
        raise ValueError(f"unsupported dtype {dtype!r} (float64 or float32)")
    return _DTYPES[key]


class Plan:
    """Compiled kernel chain for one tape.

    Keyword options mirror ``vsb_options`` (include/vsb200.h): ``dtype``
    ("float64" | "float32"), ``block`` (CTA size), ``chunk_ops`` (ops per
    chained kernel; -1 never splits), ``min_blocks``, ``maxrregcount``,
    ``smem_budget``, ``wave``, ``compile_threads``, ``verbose``, ``cache_dir``, ``team``,
    ``groups``, ``cluster``, ``outline``, ``bulk_io``, ``flags`` (``VSB_FLAG_*``: 1 paired
    cross-warp exchange, 2 split barriers, 4 shared-reciprocal division), ``tma_stages``, ``lockstep``.
    """

    def __init__(self, tape, *, dtype="float64", block=0, chunk_ops=0, min_blocks=0, maxrregcount=0,
                 smem_budget=0, wave=0, compile_threads=0, verbose=False, cache_dir=None, team=0,
                 phase_cost=0, priority=0, libdevice_trig=False, team_smem=0, groups=0, cluster=0, outline=0, bulk_io=0, flags=0,
                 tma_stages=0, lockstep=0):
        self.tape: InstructionTape = as_tape(tape)
        self.dtype_code = _dtype_code(dtype)
        self.np_dtype = np.float32 if self.dtype_code == _native.VSB_F32 else np.float64
        L = _native.lib()
        opts = Options()
        L.vsb_options_init(ctypes.byref(opts))
        opts.dtype = self.dtype_code
        opts.block = int(block)
        opts.min_blocks = int(min_blocks)
        opts.maxrregcount = int(maxrregcount)
        opts.chunk_ops = int(chunk_ops)
        opts.smem_budget = int(smem_budget)
        opts.wave = int(wave)
        opts.compile_threads = int(compile_threads)
        opts.verbose = 1 if verbose else 0
        opts.team = int(team)
        opts.phase_cost = int(phase_cost)
        opts.priority = int(priority)
        opts.libdevice_trig = 1 if libdevice_trig else 0
        opts.team_smem = int(team_smem)
        opts.groups = int(groups)
        opts.cluster = int(cluster)
        opts.outline = int(outline)
        opts.bulk_io = int(bulk_io)
        opts.flags = int(flags)
        opts.tma_stages = int(tma_stages)
        opts.lockstep = int(lockstep)
        self._cache_dir = None if cache_dir is None else str(cache_dir).encode()
        opts.cache_dir = self._cache_dir
        code, values = self.tape.packed()
        self._code = np.ascontiguousarray(code, dtype=np.int32)
        self._values = np.ascontiguousarray(values, dtype=np.float64)
        self._nnz_in = np.asarray(self.tape.nnz_in, dtype=np.int64)
        self._nnz_out = np.asarray(self.tape.nnz_out, dtype=np.int64)
        handle = ctypes.c_void_p()
        self._h = None
        check(L.vsb_plan_create(
            self._code.ctypes.data, self._values.ctypes.data, self._code.shape[0], self.tape.n_w,
            self._nnz_in.ctypes.data if self._nnz_in.size else None, len(self._nnz_in),
            self._nnz_out.ctypes.data if self._nnz_out.size else None, len(self._nnz_out),
            ctypes.byref(opts), ctypes.byref(handle)))
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _native._lib is not None:
            _native._lib.vsb_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def info(self) -> dict:
        inf = PlanInfo()
        check(_native.lib().vsb_plan_get_info(self._h, ctypes.byref(inf)))
        return inf.as_dict()

    def source(self, chunk: int = 0) -> str:
        s = ctypes.c_char_p()
        check(_native.lib().vsb_plan_source(self._h, int(chunk), ctypes.byref(s)))
        return s.value.decode()

    def cubin(self, chunk: int = 0) -> bytes:
        data, size = ctypes.c_void_p(), ctypes.c_int64()
        check(_native.lib().vsb_plan_cubin(self._h, int(chunk), ctypes.byref(data), ctypes.byref(size)))
        return ctypes.string_at(data.value, size.value) if size.value else b""

    @property
    def log(self) -> str:
        s = ctypes.c_char_p()
        check(_native.lib().vsb_plan_log(self._h, ctypes.byref(s)))
        return (s.value or b"").decode(errors="replace")

    def launches_per_eval(self, n: int) -> int:
        return int(_native.lib().vsb_launches_per_eval(self._h, int(n)))

    # -- raw entry points (pointers are ints) --------------------------------
    def eval_device(self, in_ptr, in_off, out_ptr, out_off, e0, e1, device=0, stream=0):
        in_off = np.ascontiguousarray(in_off, dtype=np.int64)
        out_off = np.ascontiguousarray(out_off, dtype=np.int64)
        check(_native.lib().vsb_eval_device(
            self._h, ctypes.c_void_p(in_ptr), in_off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            ctypes.c_void_p(out_ptr), out_off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            int(e0), int(e1), int(device), ctypes.c_void_p(stream)))

    def eval_device_ptrs(self, in_ptrs, out_ptrs, e0, e1, device=0, stream=0):
        ins = (ctypes.c_void_p * max(1, len(in_ptrs)))(*in_ptrs)
        outs = (ctypes.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        check(_native.lib().vsb_eval_device_ptrs(self._h, ins, outs, int(e0), int(e1), int(device),
                                                 ctypes.c_void_p(stream)))

    def eval_device_soa(self, in_ptrs, out_ptrs, ld, e0, e1, device=0, stream=0):
        ins = (ctypes.c_void_p * max(1, len(in_ptrs)))(*in_ptrs)
        outs = (ctypes.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        check(_native.lib().vsb_eval_device_soa(self._h, ins, outs, int(ld), int(e0), int(e1), int(device),
                                                ctypes.c_void_p(stream)))

    def rollout_device(self, state_in, state_out, in_ptrs, out_ptrs, plane, steps, e0, e1, device=0, stream=0,
                       record=True):
        """``steps`` closed-loop evaluations in one launch (``vsb_rollout_device``);
        raises ``_native.UnsupportedError`` when the plan has no such variant."""
        ins = (ctypes.c_void_p * max(1, len(in_ptrs)))(*in_ptrs)
        outs = (ctypes.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        check(_native.lib().vsb_rollout_device(self._h, int(state_in), int(state_out), ins, outs, int(plane),
                                               int(steps), int(bool(record)), int(e0), int(e1), int(device),
                                               ctypes.c_void_p(stream)))

    def prepare_rollout(self, state_in: int = 0, state_out: int = 0) -> None:
        """Compile the closed-loop variant ``rollout_device`` launches (no GPU needed);
        raises ``_native.UnsupportedError`` when the plan has none."""
        check(_native.lib().vsb_plan_prepare_rollout(self._h, int(state_in), int(state_out)))

    def eval_host(self, in_ptr, in_off, out_ptr, out_off, e0, e1, device=0):
        in_off = np.ascontiguousarray(in_off, dtype=np.int64)
        out_off = np.ascontiguousarray(out_off, dtype=np.int64)
        check(_native.lib().vsb_eval_host(
            self._h, ctypes.c_void_p(in_ptr), in_off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            ctypes.c_void_p(out_ptr), out_off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            int(e0), int(e1), int(device)))

    def eval_host_sharded(self, in_ptr, in_off, out_ptr, out_off, e0, e1, devices):
        in_off = np.ascontiguousarray(in_off, dtype=np.int64)
        out_off = np.ascontiguousarray(out_off, dtype=np.int64)
        devs = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
        check(_native.lib().vsb_eval_host_sharded(
            self._h, ctypes.c_void_p(in_ptr), in_off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            ctypes.c_void_p(out_ptr), out_off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            int(e0), int(e1), devs, len(devices)))


_CACHE: dict = {}
_CACHE_LOCK = threading.Lock()


def get_plan(tape, **opts) -> Plan:
    """Process-wide plan cache keyed by tape content + options."""
    tape = as_tape(tape)
    opts.setdefault("dtype", "float64")
    key = (tape.digest(), tuple(sorted((k, str(v)) for k, v in opts.items())))
    with _CACHE_LOCK:
        p = _CACHE.get(key)
        if p is None:
            p = Plan(tape, **opts)
            _CACHE[key] = p
        return p


def clear_plan_cache() -> None:
    with _CACHE_LOCK:
        _CACHE.clear()


def default_cache_dir() -> str:
    return os.environ.get("VSB_CACHE_DIR") or os.path.join(os.path.expanduser("~"), ".cache", "vsb200")
