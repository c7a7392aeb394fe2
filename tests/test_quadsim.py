"""Closed-loop drivers (paper_2408_09662_b200.quadsim) against goldens made by
the reference's own vecsym.quadsim (tests/golden/make_quadsim_golden.py)."""

import os

import numpy as np
import pytest

import oracle
import workloads
from paper_2408_09662_b200 import quadsim as qs

from conftest import GOLDEN, RTOL64, assert_bitwise_or_nan, assert_close


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "quadsim.npz"))


def test_params_and_theta_helpers(golden):
    p = qs.QuadParams()
    assert p.u_max == 2.0 * p.hover_thrust
    np.testing.assert_array_equal(p.vector()[[0, 1, 2, 3, 5, 13]], golden["rb_theta"][0, [0, 1, 2, 3, 5, 13]])
    assert qs.theta_index("u_max") == 4 and qs.N_THETA == 14
    with pytest.raises(ValueError):
        qs.theta_index("nope")
    with pytest.raises(ValueError):
        qs.QuadParams(mass=0.0)
    with pytest.raises(ValueError):
        qs.QuadParams(q_diag=(1.0,))
    assert qs._theta_batch(p, 3).shape == (3, 14)
    assert qs._theta_batch(p.vector()[None], 4).shape == (4, 14)
    with pytest.raises(ValueError):
        qs._as_batch(np.zeros((2, 5)), 6, "z0")
    with pytest.raises(ValueError):
        qs.rollout_batch(np.zeros((2, 6)), p, steps=0, tape=workloads.load_tape("quad_step"))
    with pytest.raises(ValueError):
        qs.roa_scan([], [0.0], [1.0], tape=workloads.load_tape("quad_step"))


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
    r1 = qs.rollout_batch(golden["rb_z0"][:5], qs.QuadParams(), steps=golden["rb_inputs"].shape[1], tape=tape)
    assert_close(r1.trajectory, golden["rb1_traj"], RTOL64 * 50, "broadcast theta")
    assert r1.batch_size == 5 and r1.steps == golden["rb_inputs"].shape[1]


@pytest.mark.gpu
def test_controls_at_matches_reference(golden):
    u = qs.controls_at(golden["rb_z0"], golden["rb_theta"], tape=workloads.load_tape("quad_step"))
    assert_close(u, golden["ca_u"], RTOL64, "controls")


@pytest.mark.gpu
def test_roa_scan_matches_reference(golden):
    masks = qs.roa_scan(golden["roa_mx"], golden["roa_mw"], golden["roa_um"], steps=200,
                        tape=workloads.load_tape("quad_step"))
    assert len(masks) == 3
    np.testing.assert_array_equal(np.stack(masks), golden["roa_masks"])


def test_csv_writers_match_reference(golden, tmp_path):
    masks = list(golden["roa_masks"])
    qs.write_roa_csv(tmp_path / "roa.csv", golden["roa_um"], golden["roa_mx"], golden["roa_mw"], masks)
    assert (tmp_path / "roa.csv").read_text() == str(golden["roa_csv"])
    rows = [("mass", float(v), int(k), *d) for v, k, d in zip(golden["ps_values"][:7], golden["ps_steps"][:7],
                                                                golden["ps_data"][:7])]
    qs.write_sweep_csv(tmp_path / "sweep.csv", rows)
    assert (tmp_path / "sweep.csv").read_text() == str(golden["sweep_csv"])
    with pytest.raises(ValueError):
        qs.write_roa_csv(tmp_path / "x.csv", [1.0, 2.0], golden["roa_mx"], golden["roa_mw"], masks[:1])


@pytest.mark.gpu
def test_param_sweep_matches_reference(golden):
    rows = qs.param_sweep("mass", [0.4, 0.5, 0.7], steps=30, tape=workloads.load_tape("quad_step"))
    assert len(rows) == golden["ps_data"].shape[0]
    assert all(r[0] == "mass" for r in rows)
    np.testing.assert_array_equal([r[1] for r in rows], golden["ps_values"])
    np.testing.assert_array_equal([r[2] for r in rows], golden["ps_steps"])
    assert_close(np.array([r[3:] for r in rows]), golden["ps_data"], RTOL64 * 50, "sweep rows")
