"""The plans the GPU tests and bench.py compile, listed so that
``__graft_entry__.build()`` can NVRTC-compile them into the in-tree cubin cache
(``.vsb_cache``, which travels to the GPU box) ahead of time.  Test
infrastructure: nothing in the product package imports this."""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def jobs() -> list[tuple]:
    """(kind, key, options) descriptors: kind "workload" (key = name) or "fuzz" (key = (family, index))."""
    from test_acceptance_fuzz import _golden, _tapes, stress_options
    from test_gpu_contract import FP32_RTOL, VARIANTS

    out = []
    z = _golden()
    for fam in ("exact", "acc"):
        for idx, tape in enumerate(_tapes(z, fam)):
            for opts in [{}] + stress_options(tape, idx):
                out.append(("fuzz", (fam, idx), opts))
    for name in ("humanoid_rbd", "ldlt_25"):
        out.append(("workload", name, {"team": 1}))
        out += [("workload", name, o) for _, o in VARIANTS]
    out += [("workload", name, {"dtype": "float32"}) for name in sorted(FP32_RTOL)]
    out += [("workload", "srbm_mpc", {"team": 8})]
    out += [("workload", "ldlt_57", {"team": 8, "groups": 2})]   # test_grouped_teams_on_the_ldlt57_solve
    for name in ("pendulum", "cartpole_rk4", "example"):
        out += [("workload", name, o) for o in ({"bulk_io": 1}, {"bulk_io": -1}, {"bulk_io": 1, "tma_stages": 3},
                                                 {"bulk_io": 1, "tma_stages": 4})]
    return out


def compile_job(job) -> str:
    from paper_2408_09662_b200 import Plan

    kind, key, opts = job
    if kind == "fuzz":
        from test_acceptance_fuzz import _golden, _tapes

        tape = _tapes(_golden(), key[0])[key[1]]
    else:
        import workloads

        tape = workloads.load_tape(key)
    Plan(tape, **opts)
    return f"{kind} {key} {opts}"
