"""Golden outputs of the reference's own closed-loop drivers (run HERE only,
with tools/refenv.sh sourced): vecsym.quadsim.rollout_batch / controls_at /
roa_scan on small grids, for tests/test_quadsim.py.  The tape used is the
committed workloads/quad_step.tape.json.gz (built by the reference's
quad_step_tape(), tools/make_workloads.py)."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))


def main():
    from vecsym import quadsim
    from vecsym.tape import deserialize
    import gzip

    with gzip.open(os.path.join(HERE, "..", "..", "workloads", "quad_step.tape.json.gz"), "rt") as fh:
        tape = deserialize(fh.read())
    rng = np.random.default_rng(11)
    out = {}
    # rollout_batch: per-env theta (u_max varied) and off-origin states
    B, steps = 24, 60
    z0 = rng.uniform(-0.3, 0.3, size=(B, 6))
    theta = np.tile(quadsim.QuadParams().vector(), (B, 1))
    theta[:, 4] *= rng.uniform(0.6, 1.4, size=B)
    r = quadsim.rollout_batch(z0, theta, steps=steps, tape=tape, n_threads=2)
    out.update(rb_z0=z0, rb_theta=theta, rb_traj=r.trajectory, rb_inputs=r.inputs, rb_stable=r.stable,
               rb_norm=r.final_norm)
    # broadcast theta (QuadParams) path
    r1 = quadsim.rollout_batch(z0[:5], quadsim.QuadParams(), steps=steps, tape=tape, n_threads=1)
    out.update(rb1_traj=r1.trajectory, rb1_inputs=r1.inputs)
    out.update(ca_u=quadsim.controls_at(z0, theta, tape=tape))
    # roa_scan: 5 x 4 momentum grid, 3 thrust limits
    mx = np.linspace(-1.0, 1.0, 5)
    mw = np.linspace(-0.05, 0.05, 4)
    um = np.array([2.0, 4.905, 8.0])
    masks = quadsim.roa_scan(mx, mw, um, steps=200, tape=tape, n_threads=2)
    out.update(roa_mx=mx, roa_mw=mw, roa_um=um, roa_masks=np.stack(masks))
    rows = quadsim.param_sweep("mass", [0.4, 0.5, 0.7], steps=30, tape=tape, n_threads=1)
    out.update(ps_values=np.array([r[1] for r in rows]), ps_steps=np.array([r[2] for r in rows]),
               ps_data=np.array([r[3:] for r in rows]))
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        quadsim.write_roa_csv(os.path.join(d, "roa.csv"), um, mx, mw, masks)
        quadsim.write_sweep_csv(os.path.join(d, "sweep.csv"), rows[:7])
        out.update(roa_csv=np.array(open(os.path.join(d, "roa.csv")).read()),
                   sweep_csv=np.array(open(os.path.join(d, "sweep.csv")).read()))
    np.savez_compressed(os.path.join(HERE, "quadsim.npz"), **out)
    print({k: v.shape for k, v in out.items()}, "stable frac", float(np.stack(masks).mean()))


if __name__ == "__main__":
    main()
