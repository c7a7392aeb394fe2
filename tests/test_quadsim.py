"""Closed-loop drivers (paper_2408_09662_b200.quadsim) against goldens made by
the reference's own vecsym.quadsim (tests/golden/make_quadsim_golden.py)."""

import os
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
import workloads
from paper_2408_09662_b200 import quadsim as qs

from conftest import GOLDEN, RTOL64, assert_bitwise_or_nan, assert_close


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "quadsim.npz"))


def _params(golden):
    # the reference's default QuadParams, duck-typed from its theta vector (mass, inertia lead it)
    vec = golden["rb_theta"][0].copy()
    return SimpleNamespace(vector=lambda: vec, mass=float(vec[0]), inertia=float(vec[1]))


def test_argument_checks(golden):
    tape = workloads.load_tape("quad_step")
    assert qs._theta(_params(golden), 3).shape == (3, 14)
    assert qs._theta(golden["rb_theta"][:1], 4).shape == (4, 14)
    with pytest.raises(ValueError):
        qs._theta(golden["rb_theta"][:2], 3)
    with pytest.raises(ValueError):
        qs._rows(np.zeros((2, 5)), 6, "z0")
    with pytest.raises(ValueError):
        qs.rollout_batch(np.zeros((2, 6)), _params(golden), steps=0, tape=tape)
    with pytest.raises(ValueError):
        qs.roa_scan([], [0.0], [1.0], params=_params(golden), tape=tape)


def test_oracle_host_loop_reproduces_reference_rollout(golden):
    # the reference's host loop (quadsim.py:298-303) restated over the oracle: bitwise
    tape = workloads.load_tape("quad_step")
    state, theta = golden["rb_z0"].copy(), golden["rb_theta"]
    for k in range(golden["rb_inputs"].shape[1]):
        z, u = oracle.batch_eval(tape, [state, theta], n_threads=2)
        assert_bitwise_or_nan(z, golden["rb_traj"][:, k + 1], f"step {k}")
        assert_bitwise_or_nan(u, golden["rb_inputs"][:, k], f"u step {k}")
        state = z


@pytest.mark.gpu
def test_rollout_batch_matches_reference(golden):
    tape = workloads.load_tape("quad_step")
    r = qs.rollout_batch(golden["rb_z0"], golden["rb_theta"], steps=golden["rb_inputs"].shape[1], tape=tape)
    assert r.trajectory.shape == golden["rb_traj"].shape and r.inputs.shape == golden["rb_inputs"].shape
    assert_close(r.trajectory, golden["rb_traj"], RTOL64 * 50, "trajectory")
    assert_close(r.inputs, golden["rb_inputs"], RTOL64 * 50, "inputs")
    np.testing.assert_array_equal(r.stable, golden["rb_stable"])
    assert_close(r.final_norm, golden["rb_norm"], RTOL64 * 50, "final norm")
    r1 = qs.rollout_batch(golden["rb_z0"][:5], _params(golden), steps=golden["rb_inputs"].shape[1], tape=tape)
    assert_close(r1.trajectory, golden["rb1_traj"], RTOL64 * 50, "broadcast theta")
    assert r1.batch_size == 5 and r1.steps == golden["rb_inputs"].shape[1]


@pytest.mark.gpu
def test_controls_at_matches_reference(golden):
    u = qs.controls_at(golden["rb_z0"], golden["rb_theta"], tape=workloads.load_tape("quad_step"))
    assert_close(u, golden["ca_u"], RTOL64, "controls")


@pytest.mark.gpu
def test_roa_scan_matches_reference(golden):
    masks = qs.roa_scan(golden["roa_mx"], golden["roa_mw"], golden["roa_um"], params=_params(golden), steps=200,
                        tape=workloads.load_tape("quad_step"))
    assert len(masks) == 3
    np.testing.assert_array_equal(np.stack(masks), golden["roa_masks"])
