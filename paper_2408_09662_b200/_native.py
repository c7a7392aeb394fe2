"""ctypes binding of libvsb200.so (C ABI: include/vsb200.h).

The product path has no fallback: if the library is missing or fails to
load, every entry point raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvsb200.so")
CSRC = os.path.join(_HERE, "csrc")

VSB_OK, VSB_ERR_INVALID, VSB_ERR_COMPILE, VSB_ERR_CUDA, VSB_ERR_NOMEM, VSB_ERR_UNSUPPORTED = range(6)
VSB_F64, VSB_F32 = 0, 1

# every symbol include/vsb200.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "vsb_version", "vsb_last_error", "vsb_options_init", "vsb_plan_create", "vsb_plan_destroy",
    "vsb_plan_get_info", "vsb_plan_source", "vsb_plan_cubin", "vsb_plan_log", "vsb_eval_device", "vsb_eval_device_ptrs",
    "vsb_eval_device_soa", "vsb_rollout_device", "vsb_plan_prepare_rollout",
    "vsb_eval_host", "vsb_eval_host_sharded", "vsb_transpose", "vsb_launches_per_eval",
    "vsb_host_alloc", "vsb_host_free", "vsb_debug_read_global",
    "vsb_pipe_create", "vsb_pipe_submit", "vsb_pipe_wait", "vsb_pipe_drain", "vsb_pipe_destroy",
)


class UnsupportedError(RuntimeError):
    """The plan has no variant for the requested call (VSB_ERR_UNSUPPORTED); callers fall back."""


class NativeLibraryError(RuntimeError):
    pass


class CompileError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class Options(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("min_blocks", ctypes.c_int32),
        ("maxrregcount", ctypes.c_int32),
        ("chunk_ops", ctypes.c_int64),
        ("smem_budget", ctypes.c_int64),
        ("wave", ctypes.c_int64),
        ("compile_threads", ctypes.c_int32),
        ("verbose", ctypes.c_int32),
        ("cache_dir", ctypes.c_char_p),
        ("team", ctypes.c_int32),
        ("phase_cost", ctypes.c_int32),
        ("priority", ctypes.c_int32),
        ("libdevice_trig", ctypes.c_int32),
        ("team_smem", ctypes.c_int64),
        ("groups", ctypes.c_int32),
        ("cluster", ctypes.c_int32),
        ("outline", ctypes.c_int32),
        ("bulk_io", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("tma_stages", ctypes.c_int32),
        ("lockstep", ctypes.c_int32),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64),
        ("n_arith_rows", ctypes.c_int64),
        ("n_live_ops", ctypes.c_int64),
        ("n_chunks", ctypes.c_int64),
        ("scratch_slots", ctypes.c_int64),
        ("scratch_loads", ctypes.c_int64),
        ("scratch_stores", ctypes.c_int64),
        ("block", ctypes.c_int32),
        ("max_regs", ctypes.c_int32),
        ("max_local_bytes", ctypes.c_int64),
        ("compile_seconds", ctypes.c_double),
        ("cache_hits", ctypes.c_int32),
        ("stage_in", ctypes.c_int32),
        ("stage_out", ctypes.c_int32),
        ("team", ctypes.c_int32),
        ("phases", ctypes.c_int64),
        ("smem_slots", ctypes.c_int64),
        ("overflow_slots", ctypes.c_int64),
        ("xfers", ctypes.c_int64),
        ("est_efficiency", ctypes.c_double),
        ("groups", ctypes.c_int32),
        ("cluster", ctypes.c_int32),
        ("remote_stores", ctypes.c_int64),
        ("code_bytes", ctypes.c_int64),
        ("n_cse", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def build(force: bool = False) -> str:
    """Compile libvsb200.so in-tree with its Makefile (nvcc + g++, no GPU needed)."""
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2408_09662_b200/csrc` (there is no CPU fallback)"
        )
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    i64p = ctypes.POINTER(ctypes.c_int64)
    L.vsb_version.restype = ctypes.c_char_p
    L.vsb_last_error.restype = ctypes.c_char_p
    L.vsb_options_init.argtypes = [ctypes.POINTER(Options)]
    L.vsb_options_init.restype = None
    L.vsb_plan_create.argtypes = [vp, vp, i64, i64, vp, i32, vp, i32, ctypes.POINTER(Options), ctypes.POINTER(vp)]
    L.vsb_plan_destroy.argtypes = [vp]
    L.vsb_plan_get_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    L.vsb_plan_source.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_char_p)]
    L.vsb_plan_log.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p)]
    L.vsb_plan_cubin.argtypes = [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.vsb_eval_device.argtypes = [vp, vp, i64p, vp, i64p, i64, i64, i32, vp]
    L.vsb_eval_device_ptrs.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), i64, i64, i32, vp]
    L.vsb_eval_device_soa.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), i64, i64, i64, i32, vp]
    L.vsb_rollout_device.argtypes = [vp, i32, i32, ctypes.POINTER(vp), ctypes.POINTER(vp), i64, i64, i32, i64, i64, i32,
                                     vp]
    L.vsb_plan_prepare_rollout.argtypes = [vp, i32, i32]
    L.vsb_eval_host.argtypes = [vp, vp, i64p, vp, i64p, i64, i64, i32]
    L.vsb_eval_host_sharded.argtypes = [vp, vp, i64p, vp, i64p, i64, i64, ctypes.POINTER(i32), i32]
    L.vsb_transpose.argtypes = [vp, vp, i64, i64, i64, i64, i32, vp]
    L.vsb_launches_per_eval.argtypes = [vp, i64]
    L.vsb_launches_per_eval.restype = i64
    L.vsb_host_alloc.argtypes = [ctypes.POINTER(vp), i64]
    L.vsb_host_free.argtypes = [vp]
    L.vsb_debug_read_global.argtypes = [vp, i32, ctypes.c_char_p, i32, vp, i64]
    L.vsb_pipe_create.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    L.vsb_pipe_submit.argtypes = [vp, vp, i64p, vp, i64p, i64, i64, i64p]
    L.vsb_pipe_wait.argtypes = [vp, i64]
    L.vsb_pipe_drain.argtypes = [vp]
    L.vsb_pipe_destroy.argtypes = [vp]
    for name in EXPORTS:
        fn = getattr(L, name)
        if fn.restype is ctypes.c_int:  # default restype: status code
            fn.restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a vsb status code to a Python exception."""
    if rc == VSB_OK:
        return
    msg = (lib().vsb_last_error() or b"").decode(errors="replace")
    if rc == VSB_ERR_INVALID:
        raise ValueError(msg)
    if rc == VSB_ERR_COMPILE:
        raise CompileError(msg)
    if rc == VSB_ERR_CUDA:
        raise CudaError(msg)
    if rc == VSB_ERR_NOMEM:
        raise MemoryError(msg)
    if rc == VSB_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise RuntimeError(f"vsb error {rc}: {msg}")
