"""The north_star parity contract at the configs' own batch sizes, the fp32
tolerances per config, and every off-by-default code-generation variant.

* fp64: ``|g - r| <= 1e-12 * max(|r|, 1)`` on EVERY row of the config's batch
  (srbm_mpc, the config-3 MPC surrogate, at B=4096; humanoid_rbd, config 2, at
  B=65536; config 4's 1e6-instance sweep on 1e4 sampled rows) against the
  pinned CPU oracle (oracle/, bit-identical to the reference on the goldens).
* fp32 mode: per-workload tolerances stated in ``FP32_RTOL`` (relative to
  max(|r|, 1) against the fp64 oracle), measured with tools/fp32_probe.py
  (profiles/r2_fp32_errors.jsonl: max 3.9e-7 pendulum, 1.5e-7 cartpole, 6.7e-8 ldlt_12,
  2.9e-6 quad_step, 3.9e-5 humanoid_rbd, 1.6e-5 rbd_chain12, 1.4e-2 srbm_mpc and 1.5e-2
  unicycle_mpc -- the penalty-SQP solves amplify fp32 rounding) and set with ~3-7x headroom; the reference is
  fp64-only, so these are this build's own contract.
* variants: thread-block clusters, instance groups, paired 128-bit exchange,
  split barriers, shared-reciprocal division and lockstep clusters must not
  change a bit.
"""

import numpy as np
import pytest

import oracle
import workloads
from conftest import RTOL64, assert_bitwise_or_nan, assert_close
from paper_2408_09662_b200 import BatchWorkspace, Plan, batch_eval

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# fp32 mode: max |g32 - r64| / max(|r64|, 1) allowed per workload
FP32_RTOL = {
    "pendulum": 2e-6, "cartpole_rk4": 1e-6, "ldlt_12": 5e-7, "ldlt_25": 5e-7, "ldlt_57": 5e-7,
    "quad_step": 2e-5, "humanoid_rbd": 2e-4, "rbd_chain12": 1e-4, "srbm_mpc": 5e-2, "unicycle_mpc": 1e-1,
}


def _host_eval(tape, ins, **opts):
    ws = BatchWorkspace(tape, ins[0].shape[0])
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    batch_eval(tape, ws, plan_options=opts or None)
    return [ws.output_matrix(j).copy() for j in range(tape.n_out)]


@pytest.mark.parametrize("name, B", [("srbm_mpc", 4096), ("humanoid_rbd", 65536)])
def test_every_row_of_config_batch(name, B):
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, B, seed=31)
    ref = oracle.batch_eval(tape, ins, n_threads=8)
    got = _host_eval(tape, ins)
    for j, (g, r) in enumerate(zip(got, ref)):
        assert np.isfinite(g).all()
        assert_close(g, r, RTOL64, f"{name} B={B} out {j} (all rows)")


def test_config4_million_instances_sampled():
    from paper_2408_09662_b200 import Function

    name, B = "srbm_mpc", 1_000_000
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, B, seed=32)
    f = Function(tape)
    outs = f(*[torch.tensor(v, device="cuda") for v in ins])
    rows = np.sort(np.random.default_rng(1).choice(B, 10_000, replace=False))
    ref = oracle.batch_eval(tape, [v[rows] for v in ins], n_threads=8)
    idx = torch.tensor(rows, device="cuda")
    for j, (o, r) in enumerate(zip(outs, ref)):
        assert bool(torch.isfinite(o).all())
        assert_close(o[idx].cpu().numpy(), r, RTOL64, f"srbm 1e6 out {j} (10k sampled rows)")


@pytest.mark.parametrize("name", sorted(FP32_RTOL))
def test_fp32_mode_per_config_tolerance(name):
    from paper_2408_09662_b200 import Function

    B = {"srbm_mpc": 512, "rbd_chain12": 256, "ldlt_57": 256, "unicycle_mpc": 512}.get(name, 2048)
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, B, seed=77)
    ref = oracle.batch_eval(tape, ins, n_threads=8)
    f = Function(tape, dtype=torch.float32)
    outs = f(*[torch.tensor(v, dtype=torch.float32, device="cuda") for v in ins])
    for j, (o, r) in enumerate(zip(outs, ref)):
        assert_close(o.double().cpu().numpy(), r, FP32_RTOL[name], f"{name} fp32 out {j}")


VARIANTS = [
    ("cluster2", {"team": 8, "cluster": 2}),
    ("groups2", {"team": 8, "groups": 2}),
    ("pair", {"team": 8, "flags": 1}),
    ("split", {"team": 8, "flags": 2}),
    ("pair+split", {"team": 12, "flags": 3}),
    ("divrecip_team", {"team": 8, "flags": 4}),
    ("divrecip_thread", {"team": 1, "flags": 4}),
    ("lockstep4", {"team": 8, "lockstep": 4}),
]


@pytest.mark.parametrize("tag, opts", VARIANTS, ids=[v[0] for v in VARIANTS])
@pytest.mark.parametrize("name", ["humanoid_rbd", "ldlt_25"])
def test_codegen_variants_are_bitwise(name, tag, opts):
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, 203, seed=33)
    base = _host_eval(tape, ins, team=1)
    got = _host_eval(tape, ins, **opts)
    info = Plan(tape, **opts).info
    if "cluster" in opts:
        assert info["cluster"] == opts["cluster"] and info["remote_stores"] > 0
    if "groups" in opts:
        assert info["groups"] == opts["groups"]
    for j, (a, b) in enumerate(zip(base, got)):
        assert_bitwise_or_nan(b, a, f"{name} {tag} out {j}")


def test_unwritten_output_nonzeros_read_zero():
    # a valid tape may leave output nonzeros unwritten (tape.py:171-258 accepts it); the
    # reference's fresh workspace holds 0 there (batchrt.py:116) -- so must ours, even
    # when the device buffers are reused after holding other data
    from paper_2408_09662_b200 import InstructionTape

    rows = [[1, 0, 0, 0, -1], [6, 1, 0, 0, -1], [2, 0, 1, 2, -1], [2, 1, 0, 0, -1]]   # out0[2] = x^2, out1[0] = x
    tape = InstructionTape("holes", np.array(rows, dtype=np.int32), np.zeros(4), 2, [1], [4, 2])
    ins = [np.random.default_rng(0).normal(size=(300, 1))]
    big = workloads.load_tape("pendulum")   # fill the device workspace with other data first
    _host_eval(big, workloads.make_inputs("pendulum", 5000, seed=1))
    o0, o1 = _host_eval(tape, ins)
    assert_bitwise_or_nan(o0[:, 2], ins[0][:, 0] * ins[0][:, 0], "stored")
    assert (o0[:, [0, 1, 3]] == 0).all() and not np.signbit(o0[:, [0, 1, 3]]).any()
    assert (o1[:, 1] == 0).all() and (o1[:, 0] == ins[0][:, 0]).all()
    ref = oracle.batch_eval(tape, ins)
    assert_bitwise_or_nan(o0, ref[0], "vs oracle")


def test_grouped_teams_on_the_ldlt57_solve():
    # 8-warp teams x 2 instance groups with the refined schedule: the shape that computed wrong
    # results while lockstep points were compiled in (profiles/r2_groups_lockstep.md); every row
    # against the oracle, one wave and several
    tape = workloads.load_tape("ldlt_57")
    for B in (256, 20000):
        ins = workloads.make_inputs("ldlt_57", B, seed=11)
        ref = oracle.batch_eval(tape, ins, n_threads=8)
        got = _host_eval(tape, ins, team=8, groups=2)
        for j, (g, r) in enumerate(zip(got, ref)):
            assert_close(g, r, RTOL64, f"ldlt_57 team 8 x 2 groups B={B} out {j}")


@pytest.mark.parametrize("name, sizes, depth", [
    ("srbm_mpc", (4096, 4096, 1000, 4096, 37), 2),     # team chain; a smaller batch reuses a grown slot
    ("srbm_mpc", (4096,) * 4, 3),
    ("cartpole_rk4", (100_000, 7, 65_536, 1), 2),      # thread mode (TMA tiles, tails)
    ("humanoid_rbd", (4096, 8192, 4096), 1),           # depth 1: every batch reuses the one slot
])
def test_pipeline_matches_batch_eval_bitwise(name, sizes, depth):
    """BatchPipeline (vsb_pipe_*) with several batches in flight returns the same bits as
    the synchronous batch_eval of each workspace, and the oracle's values."""
    from paper_2408_09662_b200 import BatchPipeline

    tape = workloads.load_tape(name)
    wss, want = [], []
    for k, B in enumerate(sizes):
        ins = workloads.make_inputs(name, B, seed=400 + k)
        ws = BatchWorkspace(tape, B)
        for i, v in enumerate(ins):
            ws.set_input(i, v)
        wss.append((ws, ins))
        want.append(_host_eval(tape, ins))
    with BatchPipeline(tape, depth=depth) as pipe:
        tickets = [pipe.submit(ws) for ws, _ in wss]
        for t, (ws, ins), ref in zip(tickets, wss, want):
            got = pipe.wait(t)
            for j, (g, r) in enumerate(zip(got, ref)):
                assert_bitwise_or_nan(g.reshape(r.shape), r, f"{name} pipe depth {depth} B={ws.batch_size} out {j}")
    ws, ins = wss[0]
    ref = oracle.batch_eval(tape, [v[:256] for v in ins], n_threads=8)
    for j, r in enumerate(ref):
        assert_close(ws.output_matrix(j)[:256], r, RTOL64, f"{name} pipe vs oracle out {j}")
