"""Benchmark / parity workloads: reference-built tapes + seeded inputs.

The ``*.tape.json.gz`` files next to this module were produced by
``tools/make_workloads.py`` with the reference's own graph builders and
``flatten`` (see that script for provenance).  ``make_inputs`` draws
physically meaningful per-element inputs so
that transcendental ulp differences are not amplified by ill-conditioning.
Used by tests/, bench.py and __graft_entry__.smoke(); not product code.
"""

from __future__ import annotations

import functools
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

NAMES = (
    "example", "pendulum", "cartpole_rk4", "ldlt_12", "ldlt_25", "ldlt_57", "quad_step",
    "unicycle_mpc", "srbm_mpc", "rbd_chain12", "humanoid_rbd",
)


def tape_path(name: str) -> str:
    return os.path.join(_HERE, f"{name}.tape.json.gz")


@functools.lru_cache(maxsize=None)
def load_tape(name: str):
    from paper_2408_09662_b200.tape import load

    return load(tape_path(name))


def _ldlt_inputs(n, batch, rng):
    out_a = np.empty((batch, n * (n + 1) // 2))
    out_b = rng.normal(size=(batch, n))
    il = np.tril_indices(n)
    step = max(1, (1 << 24) // (n * n))
    for lo in range(0, batch, step):
        hi = min(batch, lo + step)
        m = rng.normal(size=(hi - lo, n, n))
        spd = m @ np.transpose(m, (0, 2, 1)) + n * np.eye(n)
        out_a[lo:hi] = spd[:, il[0], il[1]]
    return [out_a, out_b]


SRBM_MASS = 24.0
SRBM_HOVER_Z = 0.55


def _srbm_inputs(batch, rng):
    T, nx, nu = 6, 12, 6
    hover = np.zeros(nx)
    hover[2] = SRBM_HOVER_Z
    u_h = np.array([0.0, 0.0, SRBM_MASS * 9.81 / 2] * 2)
    X0 = np.concatenate([np.tile(hover, T + 1), np.tile(u_h, T + 1)])
    X0 = np.tile(X0, (batch, 1)) + rng.normal(scale=0.01, size=(batch, X0.size))
    lam0 = np.zeros((batch, nx * (T + 1)))
    x0_bar = hover + rng.normal(scale=0.05, size=(batch, nx))
    rL = np.array([0.0, 0.1, 0.0]) + rng.uniform(-0.02, 0.02, size=(batch, 3))
    rR = np.array([0.0, -0.1, 0.0]) + rng.uniform(-0.02, 0.02, size=(batch, 3))
    xref = np.tile(hover, (batch, 1))
    return [X0, lam0, x0_bar, rL, rR, xref]


def _unicycle_inputs(batch, rng):
    T, goal, dt = 16, np.array([0.8, 0.4]), 0.15
    phi = float(np.arctan2(goal[1], goal[0]))
    cruise = float(np.linalg.norm(goal)) / (T * dt)
    h = rng.uniform(-np.pi / 2, np.pi / 2, size=batch)
    st = np.zeros((batch, T + 1, 3))
    st[:, :, 0] = np.linspace(0.0, goal[0], T + 1)
    st[:, :, 1] = np.linspace(0.0, goal[1], T + 1)
    st[:, :, 2] = np.linspace(0.0, 1.0, T + 1)[None, :] * (phi - h[:, None]) + h[:, None]
    ctl = np.tile([cruise, 0.0], (batch, T + 1))
    X = np.concatenate([st.reshape(batch, -1), ctl], axis=1)
    return [X, np.zeros((batch, 3 * (T + 1))), np.column_stack([np.zeros(batch), np.zeros(batch), h])]


def _quad_inputs(batch, rng):
    mass, inertia, r_arm, g, dt = 0.5, 0.01, 0.15, 9.81, 0.02
    theta = np.array([mass, inertia, r_arm, g, 2.0 * mass * g / 2.0,
                      10.0, 10.0, 10.0, 1.0, 1.0, 1.0, 1.0, 1.0, dt])
    theta = np.tile(theta, (batch, 1)) * (1.0 + rng.uniform(-0.1, 0.1, size=(batch, theta.size)))
    z = rng.uniform(-0.5, 0.5, size=(batch, 6))
    return [z, theta]


def make_inputs(name: str, batch: int, seed: int = 0) -> list[np.ndarray]:
    """Per-element inputs, one [batch, nnz_in[i]] float64 array per input."""
    rng = np.random.default_rng(seed)
    if name == "example":
        return [rng.uniform(-3.0, 3.0, size=(batch, 1))]
    if name == "pendulum":
        return [rng.uniform(-np.pi, np.pi, size=(batch, 2)),
                np.column_stack([rng.uniform(0.0, 1.0, batch), np.full(batch, 9.81), np.full(batch, 0.01)])]
    if name == "cartpole_rk4":
        x = rng.uniform(-1.0, 1.0, size=(batch, 4))
        x[:, 1] = rng.uniform(-np.pi, np.pi, size=batch)
        u = rng.uniform(-10.0, 10.0, size=(batch, 1))
        p = np.array([1.0, 0.1, 0.5, 0.02]) * (1.0 + rng.uniform(-0.1, 0.1, size=(batch, 4)))
        return [x, u, p]
    if name.startswith("ldlt_"):
        return _ldlt_inputs(int(name.split("_")[1]), batch, rng)
    if name == "quad_step":
        return _quad_inputs(batch, rng)
    if name == "srbm_mpc":
        return _srbm_inputs(batch, rng)
    if name == "unicycle_mpc":
        return _unicycle_inputs(batch, rng)
    if name in ("rbd_chain12", "humanoid_rbd"):
        n = 12 if name == "rbd_chain12" else 24
        return [rng.uniform(-0.5, 0.5, size=(batch, n)), rng.uniform(-1.0, 1.0, size=(batch, n))]
    raise KeyError(name)
