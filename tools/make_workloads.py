"""Generate the benchmark / parity tapes with the REFERENCE's own builders.

Runs only in the dev container (it imports the read-only reference package
``vecsym`` from /root/reference; ``source tools/refenv.sh`` first).  Every
tape is built with the reference's graph core and flattened by the
reference's ``vecsym.tape.flatten`` (tape.py:293-363), then written in the
reference's own ``"vecsym-tape"`` v1 text format (tape.py:387-409), gzipped,
under ``workloads/``.  Those files are what travels to the GPU box: nothing on
the box imports the reference.

Workloads:
  example        Fig-2 (sin x + x)^2                 tests/golden/example.tape.json
  pendulum       demos/02_batched_rollouts.py:20-31
  cartpole_rk4   config 1 (Appendix A)
  ldlt_12/25/57  bench.gen_ldlt_case(n)              bench.py:98-118
  quad_step      quadsim.quad_step_tape()            quadsim.py:197-237
  unicycle_mpc   demos/03 dynamics + stage_ineq, T=16, M=3
  srbm_mpc       config 3/4 surrogate: SRBM penalty-SQP, T=6, M=1, M_inner=2
  rbd_chain12    config 5 stress: Lagrangian + symbolic AD, 12-link chain
  humanoid_rbd   config 2 surrogate: CRBA + RNEA over a 24-DOF humanoid tree

Usage:  python tools/make_workloads.py [name ...]
"""

from __future__ import annotations

import gzip
import math
import os
import sys
import time

import numpy as np

from vecsym import symcore as sc
from vecsym.symcore import MatrixExpr, SymbolicFunction, sym, vertcat, horzcat, dot
from vecsym.tape import flatten, serialize

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "workloads")

mat = MatrixExpr.from_values


def _c(v):
    return sc.constant(float(v))


# ---------------------------------------------------------------------------
def build_example():
    # Fig-2 / golden example.tape.json: (sin x + x) * (sin x + x), 5 rows, n_w = 2
    x = sym("x", 1)
    e = sc.sin(x) + x
    return SymbolicFunction("example", [x], [e * e])


def build_pendulum():
    # demos/02_batched_rollouts.py:20-31
    state = sym("state", 2)
    params = sym("params", 3)
    theta, omega = state[0], state[1]
    c, g_l, dt = params[0], params[1], params[2]
    omega_next = omega + dt * (-c * omega - g_l * sc.sin(theta))
    theta_next = theta + dt * omega_next
    energy = 0.5 * dot(state, state) + g_l * (1.0 - sc.cos(theta))
    return SymbolicFunction(
        "pendulum_step", [state, params], [vertcat([theta_next, omega_next]), energy]
    )


def build_cartpole():
    x = sym("x", 4)
    u = sym("u", 1)
    p = sym("p", 4)
    mc, mp, l, dt = p[0], p[1], p[2], p[3]
    F = u[0]
    g = 9.81

    def f(s):
        th, xd, thd = s[1], s[2], s[3]
        st, ct = sc.sin(th), sc.cos(th)
        den = mc + mp * st * st
        xdd = (F + mp * st * (l * thd * thd + g * ct)) / den
        thdd = (-F * ct - mp * l * thd * thd * ct * st - (mc + mp) * g * st) / (l * den)
        return vertcat([xd, thd, xdd, thdd])

    k1 = f(x)
    k2 = f(x + (dt * 0.5) * k1)
    k3 = f(x + (dt * 0.5) * k2)
    k4 = f(x + dt * k3)
    xn = x + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    return SymbolicFunction("cartpole_rk4", [x, u, p], [xn])


def build_ldlt(n):
    from vecsym.bench import gen_ldlt_case

    return gen_ldlt_case(n).tape


def build_quad():
    from vecsym.quadsim import quad_step_tape

    return quad_step_tape()


def build_unicycle():
    from vecsym.ocpkit import OcpSpec, SolverConfig, fixed_iteration_solver, transcribe

    DT = 0.15
    GOAL = np.array([0.8, 0.4])

    def dynamics(x, u):
        return vertcat(
            [
                x[0] + DT * u[0] * sc.cos(x[2]),
                x[1] + DT * u[0] * sc.sin(x[2]),
                x[2] + DT * u[1],
            ]
        )

    def stage_cost(x, u):
        err = x[0:2] - mat(GOAL)
        return 0.1 * dot(u, u) + 0.3 * dot(err, err)

    def terminal_cost(x, u):
        err = x[0:2] - mat(GOAL)
        return 6.0 * dot(err, err)

    def stage_ineq(x, u):
        return vertcat([u[0] - 1.0, -u[0] - 1.0])

    spec = OcpSpec(
        n_x=3, n_u=2, T=16, dynamics=dynamics, stage_cost=stage_cost,
        terminal_cost=terminal_cost, stage_ineq=stage_ineq,
    )
    nlp = transcribe(spec)
    return fixed_iteration_solver(nlp, SolverConfig(M=3), name="unicycle_mpc")


SRBM_MASS = 24.0
SRBM_DT = 0.04
SRBM_IINV = (2.0, 1.667, 2.5)
SRBM_MU = 0.7
SRBM_HOVER_Z = 0.55


def build_srbm():
    """Single-rigid-body humanoid MPC surrogate."""
    from vecsym.ocpkit import OcpSpec, SolverConfig, fixed_iteration_solver, transcribe

    m, g, dt = SRBM_MASS, 9.81, SRBM_DT
    rL = sym("rL", 3)
    rR = sym("rR", 3)
    xref = sym("xref", 12)

    def cross(a, b):
        return vertcat(
            [
                a[1] * b[2] - a[2] * b[1],
                a[2] * b[0] - a[0] * b[2],
                a[0] * b[1] - a[1] * b[0],
            ]
        )

    def dynamics(x, u):
        p, th, v, w = x[0:3], x[3:6], x[6:9], x[9:12]
        fL, fR = u[0:3], u[3:6]
        cy, sy = sc.cos(th[2]), sc.sin(th[2])

        def yaw(r):
            return vertcat([cy * r[0] - sy * r[1], sy * r[0] + cy * r[1], r[2]])

        tau = cross(yaw(rL) - p, fL) + cross(yaw(rR) - p, fR)
        acc = (fL + fR) * (1.0 / m) - mat(np.array([0.0, 0.0, g]))
        wdot = vertcat([SRBM_IINV[k] * tau[k] for k in range(3)])
        return vertcat([p + dt * v, th + dt * w, v + dt * acc, w + dt * wdot])

    def stage_cost(x, u):
        e = x - xref
        return 0.5 * dot(e, e) + 1e-4 * dot(u, u)

    def terminal_cost(x, u):
        e = x - xref
        return 5.0 * dot(e, e)

    def stage_ineq(x, u):
        rows = []
        for f in (u[0:3], u[3:6]):
            fx, fy, fz = f[0], f[1], f[2]
            rows += [
                fx - SRBM_MU * fz,
                -fx - SRBM_MU * fz,
                fy - SRBM_MU * fz,
                -fy - SRBM_MU * fz,
                -fz,
            ]
        return vertcat(rows)

    spec = OcpSpec(
        n_x=12, n_u=6, T=6, dynamics=dynamics, stage_cost=stage_cost,
        terminal_cost=terminal_cost, stage_ineq=stage_ineq, parameters=(rL, rR, xref),
    )
    nlp = transcribe(spec)
    return fixed_iteration_solver(nlp, SolverConfig(M=1, M_inner=2), name="srbm_mpc")


def _rot(axis, c, s):
    # rotation matrix about a principal axis, entries as expressions
    one, zero = _c(1.0), _c(0.0)
    if axis == 0:
        g = [[one, zero, zero], [zero, c, -s], [zero, s, c]]
    elif axis == 1:
        g = [[c, zero, s], [zero, one, zero], [-s, zero, c]]
    else:
        g = [[c, -s, zero], [s, c, zero], [zero, zero, one]]
    return vertcat([horzcat(r) for r in g])


def build_rbd_chain12():
    """Lagrangian + symbolic-AD 12-link chain (SURVEY Appendix A stress tape)."""
    n = 12
    rng = np.random.default_rng(0)
    q = sym("q", n)
    qd = sym("qd", n)
    offs = rng.uniform(-0.3, 0.3, size=(n, 3)) + np.array([0.0, 0.0, 0.3])
    coms = rng.uniform(-0.1, 0.1, size=(n, 3)) + np.array([0.0, 0.0, 0.15])
    masses = rng.uniform(0.5, 3.0, size=n)
    inert = [np.diag(rng.uniform(0.01, 0.2, size=3)) for _ in range(n)]
    grav = 9.81

    R = MatrixExpr.eye(3)
    o = mat(np.zeros(3))
    M = None
    PE = _c(0.0)
    axes_w, origins = [], []
    for i in range(n):
        ax = i % 3
        o = o + R @ mat(offs[i])
        R = R @ _rot(ax, sc.cos(q[i]), sc.sin(q[i]))
        axes_w.append(R @ mat(np.eye(3)[ax]))
        origins.append(o)
        pc = o + R @ mat(coms[i])
        Jv = horzcat(
            [
                (
                    vertcat(
                        [
                            axes_w[j][1] * (pc[2] - origins[j][2]) - axes_w[j][2] * (pc[1] - origins[j][1]),
                            axes_w[j][2] * (pc[0] - origins[j][0]) - axes_w[j][0] * (pc[2] - origins[j][2]),
                            axes_w[j][0] * (pc[1] - origins[j][1]) - axes_w[j][1] * (pc[0] - origins[j][0]),
                        ]
                    )
                    if j <= i
                    else mat(np.zeros(3))
                )
                for j in range(n)
            ]
        )
        Jw = horzcat([axes_w[j] if j <= i else mat(np.zeros(3)) for j in range(n)])
        Iw = R @ mat(inert[i]) @ R.T
        Mi = masses[i] * (Jv.T @ Jv) + Jw.T @ Iw @ Jw
        M = Mi if M is None else M + Mi
        PE = PE + masses[i] * grav * pc[2]
    Mqd = M @ qd
    dMqd_dq = sc.jacobian(Mqd, q)
    KE2 = dot(qd, Mqd)
    bias = dMqd_dq @ qd - 0.5 * sc.jacobian(KE2, q).T + sc.jacobian(PE, q).T
    return SymbolicFunction("rbd_chain12", [q, qd], [M, bias])


# ---------------------------------------------------------------------------
# config 2 surrogate: MIT-Humanoid-shaped tree, recursive CRBA + RNEA
# floating base (6) + 2 legs x 5 + 2 arms x 4 = 24 DOF
# ---------------------------------------------------------------------------

HUMANOID_LIMBS = [
    # (name, mount offset on torso, joint axes, segment offsets)
    ("leg_l", (0.0, 0.1, -0.15), (2, 0, 1, 1, 1), (0.0, 0.0, -0.05, -0.2, -0.2)),
    ("leg_r", (0.0, -0.1, -0.15), (2, 0, 1, 1, 1), (0.0, 0.0, -0.05, -0.2, -0.2)),
    ("arm_l", (0.0, 0.15, 0.2), (1, 0, 2, 1), (0.0, 0.0, -0.15, -0.15)),
    ("arm_r", (0.0, -0.15, 0.2), (1, 0, 2, 1), (0.0, 0.0, -0.15, -0.15)),
]


def build_humanoid_rbd():
    """Mass matrix (CRBA) + bias forces (RNEA) of a 24-DOF floating-base tree.

    Spatial algebra written out over the reference's symbolic core; joint
    transforms use symbolic sin/cos of q.  The floating base is a 6-DOF
    free joint expressed in body coordinates (3 translations + 3 ZYX
    rotations, each a 1-DOF link of zero mass) so that the whole tree is
    built from revolute/prismatic 1-DOF joints.
    """
    rng = np.random.default_rng(7)
    # joint list: (parent index, type 'P'|'R', axis, offset xyz, mass, com, inertia diag)
    joints = []
    for k in range(3):
        joints.append((k - 1, "P", k, (0.0, 0.0, 0.0), 0.0, (0, 0, 0), (0, 0, 0)))
    for k, ax in enumerate((2, 1, 0)):
        last = k == 2
        joints.append(
            (2 + k, "R", ax, (0.0, 0.0, 0.0),
             8.3 if last else 0.0, (0.0, 0.0, 0.05) if last else (0, 0, 0),
             (0.08, 0.07, 0.04) if last else (0, 0, 0))
        )
    torso = len(joints) - 1
    for _, mount, axes, segs in HUMANOID_LIMBS:
        parent = torso
        for k, ax in enumerate(axes):
            off = mount if k == 0 else (0.0, 0.0, segs[k])
            mass = float(rng.uniform(0.4, 1.6))
            com = tuple(float(v) for v in rng.uniform(-0.03, 0.03, 3) + np.array([0, 0, -0.06]))
            inert = tuple(float(v) for v in rng.uniform(0.002, 0.02, 3))
            joints.append((parent, "R", ax, off, mass, com, inert))
            parent = len(joints) - 1
    n = len(joints)
    assert n == 24, n
    q = sym("q", n)
    qd = sym("qd", n)

    def skew(v):
        z = _c(0.0)
        return [[z, -v[2], v[1]], [v[2], z, -v[0]], [-v[1], v[0], z]]

    def m3(a, b):
        return [[sum_e([a[i][k] * b[k][j] for k in range(3)]) for j in range(3)] for i in range(3)]

    def mv(a, v):
        return [sum_e([a[i][k] * v[k] for k in range(3)]) for i in range(3)]

    def mtv(a, v):
        return [sum_e([a[k][i] * v[k] for k in range(3)]) for i in range(3)]

    def sum_e(xs):
        acc = xs[0]
        for x in xs[1:]:
            acc = acc + x
        return acc

    def cross(a, b):
        return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

    def el(m):
        return m.element(0, 0) if isinstance(m, MatrixExpr) else m

    qs = [q[i] for i in range(n)]
    qds = [qd[i] for i in range(n)]
    zero, one = _c(0.0), _c(1.0)
    # child-from-parent transforms: rotation E (parent->child coords) and translation p (in parent)
    E, P = [], []
    for i, (par, typ, ax, off, *_rest) in enumerate(joints):
        if typ == "P":
            E.append([[one, zero, zero], [zero, one, zero], [zero, zero, one]])
            p = [_c(off[0]), _c(off[1]), _c(off[2])]
            p[ax] = p[ax] + qs[i]
            P.append(p)
        else:
            c, s = sc.cos(qs[i]), sc.sin(qs[i])
            # E = R(q)^T
            if ax == 0:
                Rm = [[one, zero, zero], [zero, c, -s], [zero, s, c]]
            elif ax == 1:
                Rm = [[c, zero, s], [zero, one, zero], [-s, zero, c]]
            else:
                Rm = [[c, -s, zero], [s, c, zero], [zero, zero, one]]
            E.append([[Rm[j][i2] for j in range(3)] for i2 in range(3)])
            P.append([_c(off[0]), _c(off[1]), _c(off[2])])

    def xform_motion(i, v):  # parent motion vector (w, v) -> child coords
        w, lv = v
        w2 = mv(E[i], w)
        lv2 = mv(E[i], [lv[k] - cross(P[i], w)[k] for k in range(3)])
        return (w2, lv2)

    def xform_force_T(i, f):  # child force (n, f) -> parent coords
        nn, ff = f
        f2 = mtv(E[i], ff)
        n2 = mtv(E[i], nn)
        n2 = [n2[k] + cross(P[i], f2)[k] for k in range(3)]
        return (n2, f2)

    def motion_subspace(i):
        typ, ax = joints[i][1], joints[i][2]
        e = [zero, zero, zero]
        e[ax] = one
        return ([zero] * 3, e) if typ == "P" else (e, [zero] * 3)

    def crm(v, u):  # motion cross product v x u
        w, lv = v
        uw, ul = u
        return (cross(w, uw), [cross(w, ul)[k] + cross(lv, uw)[k] for k in range(3)])

    def crf(v, f):  # force cross product v x* f
        w, lv = v
        nn, ff = f
        return ([cross(w, nn)[k] + cross(lv, ff)[k] for k in range(3)], cross(w, ff))

    def inertia_apply(i, v):  # spatial inertia about joint frame times motion
        mass, com, Id = joints[i][4], joints[i][5], joints[i][6]
        w, lv = v
        if mass == 0.0:
            return ([zero] * 3, [zero] * 3)
        cvec = [_c(x) for x in com]
        # f = m (v - c x w) ; n = Ic w + c x f   with Ic = I_com - m [c]^2 handled via
        f = [mass * (lv[k] - cross(cvec, w)[k]) for k in range(3)]
        nc = [Id[k] * w[k] for k in range(3)]
        nn = [nc[k] + cross(cvec, f)[k] for k in range(3)]
        return (nn, f)

    def addv(a, b):
        return ([a[0][k] + b[0][k] for k in range(3)], [a[1][k] + b[1][k] for k in range(3)])

    def scalev(a, s):
        return ([a[0][k] * s for k in range(3)], [a[1][k] * s for k in range(3)])

    def dotf(m, f):
        return sum_e([m[0][k] * f[0][k] for k in range(3)] + [m[1][k] * f[1][k] for k in range(3)])

    # RNEA for bias C(q, qd) qd + g
    Z6 = ([zero] * 3, [zero] * 3)
    vel, acc, frc = [], [], []
    a_grav = ([zero] * 3, [zero, zero, _c(9.81)])  # base accelerates up (gravity trick)
    for i in range(n):
        par = joints[i][0]
        S = motion_subspace(i)
        vJ = scalev(S, qds[i])
        vp = vel[par] if par >= 0 else Z6
        ap = acc[par] if par >= 0 else a_grav
        vi = addv(xform_motion(i, vp), vJ)
        ai = addv(xform_motion(i, ap), crm(vi, vJ))
        vel.append(vi)
        acc.append(ai)
        Iv = inertia_apply(i, vi)
        frc.append(addv(inertia_apply(i, ai), crf(vi, Iv)))
    tau = [None] * n
    for i in reversed(range(n)):
        tau[i] = dotf(motion_subspace(i), frc[i])
        par = joints[i][0]
        if par >= 0:
            frc[par] = addv(frc[par], xform_force_T(i, frc[i]))
    # CRBA: column i of M = S_j . (composite inertia of subtree(i) applied to S_i)
    Mg = [[None] * n for _ in range(n)]
    sub = [[i] for i in range(n)]
    for i in reversed(range(n)):
        par = joints[i][0]
        if par >= 0:
            sub[par] = sub[par] + sub[i]
    # motion transport down the tree: express S_i in each descendant frame
    for i in range(n):
        Si = motion_subspace(i)
        exp = {i: Si}
        for j in sorted(sub[i]):
            if j == i:
                continue
            exp[j] = xform_motion(j, exp[joints[j][0]])
        # total force at i: sum of descendant forces transported up
        forces = {j: inertia_apply(j, exp[j]) for j in sub[i]}
        for j in sorted(sub[i], reverse=True):
            if j == i:
                continue
            par = joints[j][0]
            forces[par] = addv(forces[par], xform_force_T(j, forces[j]))
        Fi = forces[i]
        Mg[i][i] = dotf(Si, Fi)
        # propagate Fi up to ancestors for off-diagonal entries
        F = Fi
        j = i
        while joints[j][0] >= 0:
            F = xform_force_T(j, F)
            j = joints[j][0]
            Mg[j][i] = dotf(motion_subspace(j), F)
            Mg[i][j] = Mg[j][i]
    for i in range(n):
        for j in range(n):
            if Mg[i][j] is None:
                Mg[i][j] = zero
    Mmat = vertcat([horzcat([el(Mg[i][j]) if isinstance(Mg[i][j], MatrixExpr) else Mg[i][j] for j in range(n)]) for i in range(n)])
    bias = vertcat([tau[i] for i in range(n)])
    return SymbolicFunction("humanoid_rbd", [q, qd], [Mmat, bias])


BUILDERS = {
    "example": build_example,
    "pendulum": build_pendulum,
    "cartpole_rk4": build_cartpole,
    "ldlt_12": lambda: build_ldlt(12),
    "ldlt_25": lambda: build_ldlt(25),
    "ldlt_57": lambda: build_ldlt(57),
    "quad_step": build_quad,
    "unicycle_mpc": build_unicycle,
    "srbm_mpc": build_srbm,
    "rbd_chain12": build_rbd_chain12,
    "humanoid_rbd": build_humanoid_rbd,
}


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for name in names or list(BUILDERS):
        t0 = time.perf_counter()
        obj = BUILDERS[name]()
        tape = obj if hasattr(obj, "packed") else flatten(obj)
        text = serialize(tape)
        path = os.path.join(OUT, f"{name}.tape.json.gz")
        with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as fh:
            fh.write(text)
        print(
            f"{name:14s} n={tape.n_instructions:7d} n_w={tape.n_w:5d} "
            f"nnz_in={tape.nnz_in} nnz_out={tape.nnz_out} "
            f"{os.path.getsize(path)/1e6:.2f} MB  {time.perf_counter()-t0:.1f}s",
            flush=True,
        )


if __name__ == "__main__":
    main(sys.argv[1:])
