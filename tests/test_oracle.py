"""The CPU oracle (oracle/vs_oracle.c) is pinned to golden vectors produced
by the reference evaluator itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import oracle
import workloads
from conftest import EXACT_OPS, assert_bitwise_or_nan
from paper_2408_09662_b200.tape import deserialize


def _ops(z):
    return sorted({k.split("__")[0] for k in z.files})


def test_oracle_single_ops_match_reference_bitwise(golden_ops):
    names = _ops(golden_ops)
    assert len(names) == 20  # every evaluable opcode (test_batchrt.py:28-30)
    for name in names:
        tape = deserialize(str(golden_ops[f"{name}__tape"]))
        x = golden_ops[f"{name}__x"]
        (got,) = oracle.batch_eval(tape, [x[:, k : k + 1] for k in range(x.shape[1])])
        assert_bitwise_or_nan(got[:, 0], golden_ops[f"{name}__y"], name)


def test_oracle_random_tapes_match_reference_bitwise(golden_random):
    n = len({k.split("__")[0] for k in golden_random.files})
    assert n == 40
    for t in range(n):
        tape = deserialize(str(golden_random[f"t{t}__tape"]))
        ins = [golden_random[f"t{t}__in{i}"] for i in range(tape.n_in)]
        for w in (1, 3):
            outs = oracle.batch_eval(tape, ins, n_threads=w)
            for j, o in enumerate(outs):
                assert_bitwise_or_nan(o, golden_random[f"t{t}__out{j}"], f"tape {t} out {j} W={w}")


@pytest.mark.parametrize("name", workloads.NAMES)
def test_oracle_workloads_match_reference_bitwise(name, golden_workloads):
    tape = workloads.load_tape(name)
    ins = [golden_workloads[f"{name}__in{i}"] for i in range(tape.n_in)]
    outs = oracle.batch_eval(tape, ins, n_threads=2)
    for j, o in enumerate(outs):
        assert_bitwise_or_nan(o, golden_workloads[f"{name}__out{j}"], f"{name} out {j}")


def test_oracle_known_answers():
    # (sin 1 + 1)^2 = 3.3910153878893637 (test_batchrt.py:120-126)
    tape = workloads.load_tape("example")
    (y,) = oracle.serial_eval(tape, [np.array([1.0])])
    assert abs(y[0] - 3.3910153878893637) < 1e-15
    # LDL^T solve of [[4,2],[2,3]] x = (6,5) -> (1,1) needs ldlt_2; use ldlt_12 on a
    # diagonal system instead: A = 2I, b = 2 -> x = 1
    t12 = workloads.load_tape("ldlt_12")
    n = 12
    A = 2.0 * np.eye(n)
    (x,) = oracle.serial_eval(t12, [A[np.tril_indices(n)], np.full(n, 2.0)])
    np.testing.assert_allclose(x, np.ones(n), rtol=0, atol=1e-14)


def test_oracle_thread_count_invariance():
    tape = workloads.load_tape("cartpole_rk4")
    ins = workloads.make_inputs("cartpole_rk4", 103, seed=3)
    ref = oracle.batch_eval(tape, ins, n_threads=1)
    for w in (2, 3, 5, 16, 64):
        got = oracle.batch_eval(tape, ins, n_threads=w)
        for g, r in zip(got, ref):
            assert_bitwise_or_nan(g, r, f"W={w}")
