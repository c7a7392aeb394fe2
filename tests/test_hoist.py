"""Loop-invariant split (hoist.split_invariant): step(varying, pre(params)) must
equal the original tape bit for bit on the oracle (CPU), for the workloads and
the reference-generated random tapes."""

import numpy as np
import pytest

import oracle
import workloads
from paper_2408_09662_b200.hoist import split_invariant
from paper_2408_09662_b200.tape import deserialize

from conftest import assert_bitwise_or_nan


def _check(tape, ins, varying):
    s = split_invariant(tape, varying)
    if s is None:
        return None
    full = oracle.batch_eval(tape, ins, n_threads=2)
    (bnd,) = oracle.batch_eval(s.pre, [ins[i] for i in s.fixed], n_threads=2)
    got = oracle.batch_eval(s.step, [ins[i] for i in s.varying] + [bnd], n_threads=2)
    assert len(got) == len(full)
    for j, (a, b) in enumerate(zip(got, full)):
        assert_bitwise_or_nan(a, b, f"{tape.name} out {j} varying {varying}")
    return s


@pytest.mark.parametrize("name", ["quad_step", "pendulum", "cartpole_rk4", "unicycle_mpc", "ldlt_12"])
def test_split_matches_full_tape(name):
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, 67, seed=5)
    for varying in [(i,) for i in range(tape.n_in)] + [tuple(range(tape.n_in))[:2]]:
        _check(tape, ins, varying)


def test_quad_step_hoists_the_lqr_synthesis():
    # 42,501 of quad_step's 42,553 arithmetic rows depend only on theta
    s = split_invariant(workloads.load_tape("quad_step"), (0,))
    assert s.hoisted_rows == 42501 and s.step_rows == 52
    assert s.step.nnz_out == workloads.load_tape("quad_step").nnz_out


def test_split_random_tapes(golden_random):
    n = len({k.split("__")[0] for k in golden_random.files})
    done = 0
    for t in range(n):
        tape = deserialize(str(golden_random[f"t{t}__tape"]))
        if tape.n_in == 0:
            continue
        ins = [golden_random[f"t{t}__in{i}"] for i in range(tape.n_in)]
        for v in range(tape.n_in):
            done += _check(tape, ins, (v,)) is not None
    assert done > 0


def test_nothing_to_hoist():
    # every row reads the varying input: no split
    tape = workloads.load_tape("example")
    assert split_invariant(tape, tuple(range(tape.n_in))) is None
    with pytest.raises(ValueError):
        split_invariant(tape, (tape.n_in,))
