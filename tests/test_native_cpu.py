"""Host-side checks of the C ABI and the code generator that need no GPU:
the library loads and exports every declared symbol, NVRTC compiles the
generated sm_100a kernels, and the emitted code has the promised shape."""

import ctypes
import os
import re

import numpy as np
import pytest

import workloads
from paper_2408_09662_b200 import BatchWorkspace, InstructionTape, Plan, batch_eval, default_thread_count
from paper_2408_09662_b200 import _native

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "vsb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char \*)\s*\*?\s*(vsb_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_native.EXPORTS)
    assert b"sm_100a" in L.vsb_version()


def test_library_has_sm100a_code():
    so = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in so  # nvcc-built static kernels (kernels.cu)


def test_plan_errors_are_value_errors():
    # C-side validation (the reference's run_range does none: boundscheck=False)
    L = _native.lib()
    code = np.array([[4, 0, 0, 1, -1]], dtype=np.int32)  # ADD reads unwritten slots
    vals = np.zeros(1)
    nin = np.array([1], dtype=np.int64)
    h = ctypes.c_void_p()
    rc = L.vsb_plan_create(code.ctypes.data, vals.ctypes.data, 1, 2, nin.ctypes.data, 1, nin.ctypes.data, 1,
                           None, ctypes.byref(h))
    assert rc == _native.VSB_ERR_INVALID
    assert b"instruction 0: work slot read before any write" in L.vsb_last_error()


@pytest.mark.parametrize("name", ["example", "pendulum", "cartpole_rk4", "ldlt_12"])
def test_nvrtc_compiles_workload_for_sm100a(name, tmp_path):
    p = Plan(workloads.load_tape(name), cache_dir=str(tmp_path), verbose=True)
    info = p.info
    assert info["n_chunks"] == 1 and info["scratch_slots"] == 0
    # at most a few spilled registers on the small tapes (they are compiled for 8 CTAs/SM =
    # 64 registers, which measured faster than spill-free 96 registers: cartpole 0.076 vs 0.096 ms)
    assert info["max_local_bytes"] <= 128
    src = p.source(0)
    assert "work[" not in src               # no global work vector (codegen.py:29-56 shape is gone)
    assert "fmin(" not in src.replace("vs_fmin(", "")  # select-based min/max only
    assert "sm_100a" in p.log
    # cache hit on the second build
    q = Plan(workloads.load_tape(name), cache_dir=str(tmp_path))
    assert q.info["cache_hits"] == 1 and q.info["compile_seconds"] == 0.0


def test_ssa_drops_dead_code_and_assign():
    rows = [
        [1, 0, 0, 0, -1],   # x
        [13, 1, 0, -1, -1], # SQ  (dead: overwritten before use)
        [3, 1, 0, -1, -1],  # ASSIGN w1 = w0 (alias, no instruction)
        [14, 0, 1, -1, -1], # SIN
        [2, 0, 0, 0, -1],
    ]
    t = InstructionTape("dce", np.array(rows, dtype=np.int32), np.zeros(5), 2, [1], [1])
    p = Plan(t, cache_dir="")
    src = p.source(0)
    body = src.split("srow = ")[1]
    assert "v0 * v0" not in body and "sin(v0)" in body  # SQ eliminated, ASSIGN aliased
    assert p.info["n_live_ops"] == 1 and p.info["n_arith_rows"] == 2


def test_splitter_cuts_large_tapes_and_bounds_liveness():
    t = workloads.load_tape("quad_step")
    p = Plan(t, cache_dir="", chunk_ops=6000)
    info = p.info
    assert info["n_chunks"] >= 6
    assert 0 < info["scratch_slots"] <= t.n_w + 100
    srcs = [p.source(c) for c in range(info["n_chunks"])]
    assert all("S[" in s for s in srcs)
    assert p.launches_per_eval(4096) == info["n_chunks"]


def test_workspace_contract_without_gpu():
    t = workloads.load_tape("pendulum")
    ws = BatchWorkspace(t, 17)
    assert [v.shape for v in ws.inputs] == [(34,), (51,)]
    assert [v.shape for v in ws.outputs] == [(34,), (17,)]
    assert ws.work.shape == (17 * t.n_w,)
    bufs = list(ws.inputs) + [ws.work] + list(ws.outputs)
    for i in range(len(bufs)):
        for j in range(i + 1, len(bufs)):
            assert not np.shares_memory(bufs[i], bufs[j])
    ws.input_matrix(0)[:, 0] = np.arange(17)
    assert ws.inputs[0][::2].tolist() == list(range(17))
    with pytest.raises(ValueError, match="expected 2 values, got 3"):
        ws.set_input(0, np.zeros(3))
    with pytest.raises(ValueError, match=r"expected shape \(17, 3\)"):
        ws.set_input(1, np.zeros((2, 3)))
    with pytest.raises(ValueError, match="batch_size must be >= 1"):
        BatchWorkspace(t, 0)
    with pytest.raises(ValueError, match="workspace/tape mismatch"):
        batch_eval(workloads.load_tape("example"), ws)
    with pytest.raises(ValueError, match="n_threads must be >= 1"):
        batch_eval(t, ws, n_threads=0)


def test_thread_count_env_override(monkeypatch):
    monkeypatch.setenv("VECSYM_THREADS", "3")
    assert default_thread_count() == 3
    for bad in ("zero", "0"):
        monkeypatch.setenv("VECSYM_THREADS", bad)
        with pytest.raises(ValueError, match="VECSYM_THREADS"):
            default_thread_count()
    monkeypatch.delenv("VECSYM_THREADS")
    assert default_thread_count() == (os.cpu_count() or 1)


def test_auto_team_width_follows_the_scheduled_live_set():
    # >= 40k-op tapes: 16 warps unless the register live set at 16 warps is past the
    # register file (measured in profiles/r1_sweeps_r50_team_width.jsonl)
    want = {"srbm_mpc": 16, "ldlt_57": 12, "rbd_chain12": 8, "humanoid_rbd": 12, "pendulum": 0}
    for name, team in want.items():
        p = Plan(workloads.load_tape(name), cache_dir="", compile_threads=-1)
        assert p.info["team"] == team, name


def test_rollout_device_argument_errors_without_gpu():
    # vsb_rollout_device validates before touching the device (ValueError like the reference)
    plan = Plan(workloads.load_tape("pendulum"), compile_threads=-1)
    ptrs = [0] * 2
    with pytest.raises(ValueError, match="out of range"):
        plan.rollout_device(5, 0, ptrs, ptrs, 10, 3, 0, 10)
    with pytest.raises(ValueError, match="sizes differ"):
        plan.rollout_device(1, 1, ptrs, ptrs, 10, 3, 0, 10)   # 3 parameters vs 1 energy output
    with pytest.raises(ValueError, match="plane"):
        plan.rollout_device(0, 0, ptrs, ptrs, 5, 3, 0, 10)


def test_hoisted_split_is_memoised():
    from paper_2408_09662_b200 import rollout

    t = workloads.load_tape("quad_step")
    a = rollout._split_of(t, 0)
    assert rollout._split_of(workloads.load_tape("quad_step"), 0) is a
    assert a.hoisted_rows == 42501


def test_value_numbering_merges_only_exact_equivalences():
    # exact GVN + IEEE identities (codegen.cpp build_program): counted without compiling
    from vn_tapes import EXPECTED_CSE, vn_tape

    p = Plan(vn_tape(), cache_dir="", compile_threads=-1)
    assert p.info["n_cse"] == EXPECTED_CSE
    # 16 arithmetic rows - 10 merged = 6 live ops: NEG x, x+y, x*y, fmin(x,y), fmin(y,x), x+0
    assert p.info["n_live_ops"] == 6


@pytest.mark.parametrize("prio", [0, 1])
def test_refined_team_schedules_compile(prio, tmp_path):
    # the local search (refine_schedule) moves ops between warps and phases; every
    # same-warp consumer must still follow its producer in the emitted code (a violation
    # surfaces as an NVRTC redeclaration error).  Critical-path priority (prio=1) leaves the
    # greedy warp-phase order far from program order -- the case that exposed it.
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from test_acceptance_fuzz import _golden, _tapes

    tapes = _tapes(_golden(), "exact")
    for idx in (40, 77, 95):
        p = Plan(tapes[idx], team=8, priority=prio, cache_dir=str(tmp_path))
        assert p.info["team"] == 8 and p.info["n_chunks"] >= 1


def test_pipeline_argument_errors_without_gpu():
    """BatchPipeline / vsb_pipe_* reject bad arguments before touching a device."""
    import ctypes

    from paper_2408_09662_b200 import BatchPipeline, _native

    t = workloads.load_tape("pendulum")
    with pytest.raises(ValueError, match="depth must be in"):
        BatchPipeline(t, depth=0)
    pipe = BatchPipeline(t)
    with pytest.raises(ValueError, match="workspace/tape mismatch"):
        pipe.submit(BatchWorkspace(workloads.load_tape("example"), 3))
    with pytest.raises(ValueError, match="unknown or already waited ticket"):
        pipe.wait(0)
    L = _native.lib()
    h = ctypes.c_void_p()
    with pytest.raises(ValueError, match="depth"):
        _native.check(L.vsb_pipe_create(vsb_plan_handle(t), 0, 0, ctypes.byref(h)))
    for rc in (L.vsb_pipe_submit(None, None, None, None, None, 0, 1, None), L.vsb_pipe_wait(None, 0),
               L.vsb_pipe_drain(None)):
        with pytest.raises(ValueError, match="null pipe"):
            _native.check(rc)


def vsb_plan_handle(tape):
    from paper_2408_09662_b200 import get_plan

    return get_plan(tape).handle
