"""GPU parity: the sm_100a path (through the C ABI) vs the reference's own
outputs (golden vectors) and vs the CPU oracle on seeded inputs.

Contract: transcendental-free ops are bit-identical to the reference; every
result is within |g - r| <= 1e-12 * max(|r|, 1) in fp64 (BASELINE.json
north_star); NaN == NaN; infinities match exactly.
"""

import math

import numpy as np
import pytest

import oracle
import workloads
from conftest import EXACT_OPS, RTOL32, RTOL64, assert_bitwise_or_nan, assert_close, assert_parity
from paper_2408_09662_b200 import BatchWorkspace, InstructionTape, Plan, batch_eval, serial_eval
from paper_2408_09662_b200.tape import OpCode, deserialize

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def gpu_eval(tape, inputs, **plan_options):
    B = inputs[0].shape[0] if inputs else 1
    ws = BatchWorkspace(tape, B)
    for i, v in enumerate(inputs):
        ws.set_input(i, v)
    batch_eval(tape, ws, plan_options=plan_options or None)
    return [ws.output_matrix(j).copy() for j in range(tape.n_out)]


def test_cuda_present():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def test_single_ops_vs_reference(golden_ops):
    names = sorted({k.split("__")[0] for k in golden_ops.files})
    for name in names:
        tape = deserialize(str(golden_ops[f"{name}__tape"]))
        x = golden_ops[f"{name}__x"]
        (got,) = gpu_eval(tape, [x[:, k : k + 1] for k in range(x.shape[1])])
        ref = golden_ops[f"{name}__y"]
        if name in EXACT_OPS:
            assert_bitwise_or_nan(got[:, 0], ref, name)
        else:
            # libdevice vs glibc: within the fp64 contract on the whole SPECIALS grid
            assert_close(got[:, 0], ref, RTOL64, name)


def test_random_tapes_vs_reference(golden_random):
    n = len({k.split("__")[0] for k in golden_random.files})
    for t in range(n):
        tape = deserialize(str(golden_random[f"t{t}__tape"]))
        ins = [golden_random[f"t{t}__in{i}"] for i in range(tape.n_in)]
        outs = gpu_eval(tape, ins)
        # random tapes compose tan/pow/exp/step on unbounded values; the bound is
        # 1e-12 or the reference's own spread under a 1-ulp libm change
        base, spread = oracle.sensitivity(tape, ins)
        for j, o in enumerate(outs):
            assert_bitwise_or_nan(base[j], golden_random[f"t{t}__out{j}"], f"oracle tape {t}")
            assert_parity(o, golden_random[f"t{t}__out{j}"], spread[j], what=f"tape {t} out {j}")


@pytest.mark.parametrize("name", workloads.NAMES)
def test_workloads_vs_reference(name, golden_workloads):
    tape = workloads.load_tape(name)
    ins = [golden_workloads[f"{name}__in{i}"] for i in range(tape.n_in)]
    outs = gpu_eval(tape, ins)
    for j, o in enumerate(outs):
        # the strict north_star contract on every workload: 1e-12 relative to max(|r|, 1)
        assert_close(o, golden_workloads[f"{name}__out{j}"], RTOL64, f"{name} out {j}")


@pytest.mark.parametrize("name, team", [("cartpole_rk4", 4), ("quad_step", 16), ("humanoid_rbd", 8),
                                        ("ldlt_25", 16), ("ldlt_12", 2), ("unicycle_mpc", 8)])
def test_team_mode_equals_thread_mode_bitwise(name, team):
    # intra-instance parallel kernels compute exactly the same IEEE operations
    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, 203, seed=11)
    one = gpu_eval(tape, ins, team=1)
    many = gpu_eval(tape, ins, team=team)
    for a, b in zip(one, many):
        assert_bitwise_or_nan(a, b, f"{name} team={team}")


def test_team_mode_srbm_vs_oracle():
    tape = workloads.load_tape("srbm_mpc")
    ins = workloads.make_inputs("srbm_mpc", 100, seed=12)
    base = oracle.batch_eval(tape, ins, n_threads=4)
    got = gpu_eval(tape, ins, team=8)
    for j, (g, r) in enumerate(zip(got, base)):
        assert_close(g, r, RTOL64, f"srbm team=8 out {j}")


def test_transcendental_free_workload_is_bitwise():
    # ldlt_12 uses only + - * / and selects: bit-identical to the reference CPU path
    tape = workloads.load_tape("ldlt_12")
    ins = workloads.make_inputs("ldlt_12", 1000, seed=9)
    ref = oracle.batch_eval(tape, ins, n_threads=4)
    got = gpu_eval(tape, ins)
    for g, r in zip(got, ref):
        assert_bitwise_or_nan(g, r, "ldlt_12")


def test_known_answer_fig2():
    tape = workloads.load_tape("example")
    (y,) = serial_eval(tape, [np.array([1.0])])
    assert y.tolist() == [(math.sin(1.0) + 1.0) ** 2]
    assert abs(y[0] - 3.3910153878893637) < 1e-15


@pytest.mark.parametrize("B", [1, 2, 31, 103, 129, 4097])
def test_ragged_batches(B):
    tape = workloads.load_tape("cartpole_rk4")
    ins = workloads.make_inputs("cartpole_rk4", B, seed=B)
    ref = oracle.batch_eval(tape, ins)
    got = gpu_eval(tape, ins)
    for g, r in zip(got, ref):
        assert_close(g, r, RTOL64, f"B={B}")


def test_chunked_equals_single_kernel():
    # forcing the kernel splitter must not change a single bit
    tape = workloads.load_tape("ldlt_25")
    ins = workloads.make_inputs("ldlt_25", 300, seed=1)
    one = gpu_eval(tape, ins, chunk_ops=-1)
    many = gpu_eval(tape, ins, chunk_ops=700)
    assert Plan(tape, chunk_ops=700).info["n_chunks"] > 5
    for a, b in zip(one, many):
        assert_bitwise_or_nan(a, b, "chunked")


@pytest.mark.parametrize("block", [32, 64, 256])
def test_block_size_invariance(block):
    tape = workloads.load_tape("quad_step")
    ins = workloads.make_inputs("quad_step", 777, seed=2)
    ref = gpu_eval(tape, ins, team=1)
    got = gpu_eval(tape, ins, team=1, block=block)
    for a, b in zip(ref, got):
        assert_bitwise_or_nan(a, b, f"block={block}")


def test_constant_only_tape():
    # n_in = 0 (test_batchrt.py:265-272): 2.5 + 0.75 = 3.25 for every element
    code = np.array([[0, 0, -1, -1, -1], [0, 1, -1, -1, -1], [4, 0, 0, 1, -1], [2, 0, 0, 0, -1]], dtype=np.int32)
    tape = InstructionTape("k", code, [2.5, 0.75, 0.0, 0.0], 2, [], [1])
    ws = BatchWorkspace(tape, 9)
    batch_eval(tape, ws, n_threads=2)
    assert ws.outputs[0].tolist() == [3.25] * 9


def test_interleaved_rows_and_overwritten_outputs():
    # valid tapes may interleave INPUT/OUTPUT rows, store a slot twice, and
    # overwrite a slot after storing it (tape.py:171-258 allows all of it)
    rows = [
        [1, 0, 0, 0, -1],   # w0 = x[0]
        [2, 0, 0, 1, -1],   # out0[1] = w0          (later overwritten)
        [1, 1, 0, 1, -1],   # w1 = x[1]
        [6, 0, 0, 1, -1],   # w0 = w0 * w1
        [2, 0, 0, 0, -1],   # out0[0] = w0
        [8, 1, 0, -1, -1],  # w1 = -w0
        [2, 0, 1, 1, -1],   # out0[1] = w1          (last store wins)
        [2, 1, 1, 0, -1],   # out1[0] = w1
    ]
    tape = InstructionTape("mix", np.array(rows, dtype=np.int32), np.zeros(len(rows)), 2, [2], [2, 1])
    ins = [np.random.default_rng(0).normal(size=(50, 2))]
    ref = oracle.batch_eval(tape, ins)
    got = gpu_eval(tape, ins)
    for g, r in zip(got, ref):
        assert_bitwise_or_nan(g, r, "interleaved")


def test_device_subrange_matches_full():
    # vsb_eval_device over [e0, e1) of a device workspace == that slice of a full run
    tape = workloads.load_tape("pendulum")
    B = 1000
    ins = workloads.make_inputs("pendulum", B, seed=4)
    ref = oracle.batch_eval(tape, ins)
    plan = Plan(tape)
    nin, nout = tape.nnz_in, tape.nnz_out
    in_off = np.concatenate([[0], np.cumsum(np.array(nin) * B)])
    out_off = np.concatenate([[0], np.cumsum(np.array(nout) * B)])
    d_in = torch.tensor(np.concatenate([v.ravel() for v in ins]), device="cuda")
    d_out = torch.full((int(out_off[-1]),), float("nan"), dtype=torch.float64, device="cuda")
    for e0, e1 in [(0, 333), (333, 334), (334, 1000)]:
        plan.eval_device(d_in.data_ptr(), in_off, d_out.data_ptr(), out_off, e0, e1, 0,
                         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    out = d_out.cpu().numpy()
    for j in range(tape.n_out):
        assert_close(out[out_off[j] : out_off[j + 1]].reshape(B, nout[j]), ref[j], RTOL64, "subrange")


def test_torch_function_aos_and_soa():
    from paper_2408_09662_b200 import Function

    tape = workloads.load_tape("cartpole_rk4")
    B = 5000
    ins = workloads.make_inputs("cartpole_rk4", B, seed=5)
    ref = oracle.batch_eval(tape, ins, n_threads=4)
    f = Function(tape)
    outs = f(*[torch.tensor(v, device="cuda") for v in ins])
    assert_close(outs[0].cpu().numpy(), ref[0], RTOL64, "aos")
    fs = Function(tape, layout="soa")
    outs = fs(*[torch.tensor(v.T.copy(), device="cuda") for v in ins])
    assert_close(outs[0].cpu().numpy().T, ref[0], RTOL64, "soa")
    assert f(*[torch.empty((0, nz), dtype=torch.float64, device="cuda") for nz in tape.nnz_in])[0].shape == (0, 4)


def test_fp32_mode_within_stated_tolerance():
    from paper_2408_09662_b200 import Function

    tape = workloads.load_tape("cartpole_rk4")
    ins = workloads.make_inputs("cartpole_rk4", 4096, seed=6)
    ref = oracle.batch_eval(tape, ins)
    f = Function(tape, dtype=torch.float32)
    (o,) = f(*[torch.tensor(v, dtype=torch.float32, device="cuda") for v in ins])
    assert_close(o.double().cpu().numpy(), ref[0], RTOL32, "fp32")


def test_large_batch_properties():
    # B = 1e6 (config 1/4 scale): spot-check rows against the oracle and check
    # that the kernel is a pure function of each row (permutation equivariance)
    from paper_2408_09662_b200 import Function

    tape = workloads.load_tape("cartpole_rk4")
    B = 1_000_000
    ins = workloads.make_inputs("cartpole_rk4", B, seed=7)
    f = Function(tape)
    dins = [torch.tensor(v, device="cuda") for v in ins]
    (o,) = f(*dins)
    rows = np.random.default_rng(0).choice(B, 2000, replace=False)
    ref = oracle.batch_eval(tape, [v[rows] for v in ins])
    assert_close(o[torch.tensor(rows, device="cuda")].cpu().numpy(), ref[0], RTOL64, "sample")
    perm = torch.randperm(B, device="cuda")
    (op,) = f(*[x[perm] for x in dins])
    assert torch.equal(op, o[perm])
    assert torch.isfinite(o).all()


def test_multi_device_sharder_single_gpu():
    # the sharder over a device list (here [0, 0]) must equal one-device evaluation
    tape = workloads.load_tape("quad_step")
    ins = workloads.make_inputs("quad_step", 1001, seed=8)
    ws = BatchWorkspace(tape, 1001)
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    batch_eval(tape, ws, devices=[0, 0])
    sharded = [ws.output_matrix(j).copy() for j in range(tape.n_out)]
    single = gpu_eval(tape, ins)
    for a, b in zip(sharded, single):
        assert_bitwise_or_nan(a, b, "sharded")


@pytest.mark.parametrize("name, steps", [("pendulum", 50), ("quad_step", 20)])
def test_device_rollout_matches_host_loop(name, steps):
    # quadsim.rollout_batch's host loop (quadsim.py:298-303) vs the captured device loop
    from paper_2408_09662_b200.rollout import rollout

    tape = workloads.load_tape(name)
    B = 500
    ins = workloads.make_inputs(name, B, seed=21)
    traj, outs = rollout(tape, torch.tensor(ins[0], device="cuda"), [None] + [torch.tensor(v, device="cuda")
                                                                             for v in ins[1:]], steps)
    traj = traj.cpu().numpy()
    state = ins[0].copy()
    for k in range(steps):
        res = oracle.batch_eval(tape, [state] + ins[1:], n_threads=4)
        # trajectories of a well-conditioned map: 1-ulp libm differences may
        # accumulate linearly over the steps
        assert_close(traj[:, k + 1], res[0], RTOL64 * 50, f"{name} step {k}")
        for j, o in outs.items():
            assert_close(o[:, k].cpu().numpy(), res[j], RTOL64 * 50, f"{name} step {k} out {j}")
        state = res[0]


@pytest.mark.parametrize("name", ["quad_step", "cartpole_rk4", "unicycle_mpc"])
def test_hoisted_rollout_equals_unhoisted(name):
    # loop-invariant rows evaluated once (hoist.split_invariant) == every step, bit for bit
    from paper_2408_09662_b200.rollout import Rollout

    tape = workloads.load_tape(name)
    B, steps = 300, 8
    ins = workloads.make_inputs(name, B, seed=23)
    res = []
    for hoist in (True, False):
        r = Rollout(tape, B, steps, hoist=hoist)
        assert (r.split is not None) == hoist
        r.set(torch.tensor(ins[0], device="cuda"), [torch.tensor(v, device="cuda") for v in ins[1:]])
        traj, outs = r.run()
        res.append((traj.cpu().numpy(), {j: o.cpu().numpy() for j, o in outs.items()}))
    assert_bitwise_or_nan(res[0][0], res[1][0], f"{name} traj")
    for j in res[1][1]:
        assert_bitwise_or_nan(res[0][1][j], res[1][1][j], f"{name} out {j}")


@pytest.mark.parametrize("name", ["pendulum", "quad_step"])
@pytest.mark.parametrize("fused", [None, False])
def test_rollout_without_trajectory(name, fused):
    # roa_scan's mode (quadsim.py:363-369): only the final state is kept; same bits as
    # the recorded trajectory's last plane
    from paper_2408_09662_b200.rollout import Rollout

    tape = workloads.load_tape(name)
    B, steps = 777, 9
    ins = workloads.make_inputs(name, B, seed=37)
    finals = []
    for record in (True, False):
        r = Rollout(tape, B, steps, record=record, fused=fused)
        r.set(torch.tensor(ins[0], device="cuda"), [torch.tensor(v, device="cuda") for v in ins[1:]])
        traj, outs = r.run()
        assert fused is not None or r.fused
        if not record:
            assert traj.shape[0] == 2 and not outs
            assert_bitwise_or_nan(traj[0].cpu().numpy(), ins[0], "initial state kept")
        finals.append(traj[-1].cpu().numpy())
    assert_bitwise_or_nan(finals[1], finals[0], f"{name} final state")


@pytest.mark.parametrize("name", ["pendulum", "quad_step"])
def test_fp32_rollout_fused_equals_loop(name):
    from paper_2408_09662_b200.rollout import Rollout

    tape = workloads.load_tape(name)
    B, steps = 513, 7
    ins = workloads.make_inputs(name, B, seed=41)
    res = []
    for fused in (None, False):
        r = Rollout(tape, B, steps, fused=fused, dtype="float32")
        assert r.traj.dtype == torch.float32
        r.set(torch.tensor(ins[0], device="cuda"), [torch.tensor(v, device="cuda") for v in ins[1:]])
        traj, _ = r.run()
        res.append(traj.cpu().numpy())
    assert_bitwise_or_nan(res[0], res[1], f"{name} fp32 traj")
    assert np.abs(res[0][1] - ins[0]).max() < 10.0   # one step stays near the start


@pytest.mark.parametrize("distinct", [1, 3])
def test_rollout_dedup_of_parameter_rows(distinct):
    # rollout_batch broadcasts one theta, roa_scan has one per thrust limit: the hoisted
    # pre tape runs once per distinct row (by bit pattern) and is gathered -- bitwise the same
    from paper_2408_09662_b200.rollout import Rollout

    tape = workloads.load_tape("quad_step")
    B, steps = 600, 10
    ins = workloads.make_inputs("quad_step", B, seed=31)
    theta = np.repeat(ins[1][:1], B, axis=0)
    if distinct == 3:
        # rows 3k / 3k+1 differ only in the sign of a zero: distinct by bit pattern
        theta[0::3, 0] = 0.0
        theta[1::3, 0] = -0.0
        theta[2::3] = ins[1][1]
    res = []
    for dedup in (None, False):
        r = Rollout(tape, B, steps, dedup=dedup)
        r.set(torch.tensor(ins[0], device="cuda"), [torch.tensor(theta, device="cuda")])
        traj, outs = r.run()
        if dedup is None:
            assert r.u_count == distinct
        res.append((traj.cpu().numpy(), {j: o.cpu().numpy() for j, o in outs.items()}))
        r.set(torch.tensor(ins[0], device="cuda"), [torch.tensor(theta, device="cuda")])  # re-set keeps the graph
        traj2, _ = r.run()
        assert_bitwise_or_nan(traj2.cpu().numpy(), res[-1][0], "re-run")
    assert_bitwise_or_nan(res[0][0], res[1][0], "traj")
    for j in res[1][1]:
        assert_bitwise_or_nan(res[0][1][j], res[1][1][j], f"out {j}")


@pytest.mark.parametrize("name, hoist, expect_fused", [("pendulum", False, True), ("cartpole_rk4", False, True),
                                                       ("quad_step", True, True), ("quad_step", False, False)])
@pytest.mark.parametrize("B", [1, 129, 3000])
def test_fused_rollout_kernel_equals_step_loop(name, hoist, expect_fused, B):
    # one closed-loop launch (state in registers, vsb_rollout_device) == K chained evaluations, bitwise
    from paper_2408_09662_b200.rollout import Rollout

    tape = workloads.load_tape(name)
    steps = 12
    ins = workloads.make_inputs(name, B, seed=29)
    res = []
    for fused in (True, False):
        r = Rollout(tape, B, steps, hoist=hoist, fused=fused, use_graph=False)
        r.set(torch.tensor(ins[0], device="cuda"), [torch.tensor(v, device="cuda") for v in ins[1:]])
        traj, outs = r.run()
        if fused:
            # team-mode (multi-warp) plans fall back to the step loop
            assert r.fused == expect_fused
            if expect_fused:
                assert r.launches_per_run == 1 + (r.pre_plan.launches_per_eval(B) if hoist else 0)
        res.append((traj.cpu().numpy(), {j: o.cpu().numpy() for j, o in outs.items()}, r.fused))
    assert res[1][2] is False
    assert_bitwise_or_nan(res[0][0], res[1][0], f"{name} traj")
    for j in res[1][1]:
        assert_bitwise_or_nan(res[0][1][j], res[1][1][j], f"{name} out {j}")


@pytest.mark.parametrize("name", ["pendulum", "cartpole_rk4", "example"])
@pytest.mark.parametrize("B", [1, 127, 128, 129, 1000, 4103, 65536])
def test_tma_tile_pipeline_equals_classic_kernel(name, B):
    # persistent cp.async.bulk tile pipeline (full 128-instance tiles) + classic tail ==
    # classic staged kernel, bit for bit, and both match the oracle
    import torch

    import paper_2408_09662_b200 as vsb

    tape = workloads.load_tape(name)
    ins = workloads.make_inputs(name, B, seed=B + 5)
    xs = [torch.tensor(v, device="cuda") for v in ins]
    fast = vsb.Function(tape, bulk_io=1)(*xs)       # force the TMA kernel at every size
    plain = vsb.Function(tape, bulk_io=-1)(*xs)
    assert vsb.get_plan(tape, bulk_io=1).info["n_chunks"] == 1
    for a, b in zip(fast, plain):
        assert_bitwise_or_nan(a.cpu().numpy(), b.cpu().numpy(), f"{name} B={B}")
    for stages in (3, 4):                           # deeper tile pipelines
        deep = vsb.Function(tape, bulk_io=1, tma_stages=stages)(*xs)
        for a, b in zip(deep, plain):
            assert_bitwise_or_nan(a.cpu().numpy(), b.cpu().numpy(), f"{name} B={B} stages={stages}")
    if B <= 4103:
        ref = oracle.batch_eval(tape, ins)
        for a, r in zip(fast, ref):
            assert_close(a.cpu().numpy(), r, RTOL64, f"{name} B={B}")


@pytest.mark.parametrize("name", ["cartpole_rk4", "ldlt_12", "srbm_mpc"])
def test_batch_equals_serial_bitwise(name):
    # test_batchrt.py:163-200: a batch row is bit-identical to serial_eval of that row
    # (thread, TMA and team kernels alike)
    tape = workloads.load_tape(name)
    B = 4096 if name != "srbm_mpc" else 256
    ins = workloads.make_inputs(name, B, seed=21)
    batch = gpu_eval(tape, ins)
    for row in (0, 1, B // 2, B - 1):
        one = serial_eval(tape, [v[row] for v in ins])
        for j, o in enumerate(one):
            assert_bitwise_or_nan(batch[j][row], o, f"{name} row {row} out {j}")


@pytest.mark.parametrize("name, team", [("cartpole_rk4", 0), ("humanoid_rbd", 0), ("srbm_mpc", 16)])
def test_element_order_shuffling(name, team):
    # test_batchrt.py:224-262: permuting the batch permutes the outputs, bit for bit
    tape = workloads.load_tape(name)
    B = 1000 if name != "srbm_mpc" else 300
    ins = workloads.make_inputs(name, B, seed=22)
    perm = np.random.default_rng(3).permutation(B)
    opts = {"team": team} if team else {}
    a = gpu_eval(tape, ins, **opts)
    b = gpu_eval(tape, [v[perm] for v in ins], **opts)
    for x, y in zip(a, b):
        assert_bitwise_or_nan(x[perm], y, f"{name} permuted")


def test_nan_and_inf_inputs_propagate_like_the_reference():
    # test_batchrt.py:84-117 at tape level: non-finite inputs flow through sin/cos/div the
    # same way (NaN == NaN, infinities exact)
    tape = workloads.load_tape("cartpole_rk4")
    ins = workloads.make_inputs("cartpole_rk4", 256, seed=23)
    specials = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1e308, -1e308, 5e-324]
    for k, v in enumerate(specials):
        ins[0][k * 4 % 256, k % 4] = v
        ins[2][(k * 7 + 1) % 256, k % 4] = v
    ref = oracle.batch_eval(tape, ins)
    got = gpu_eval(tape, ins)
    for g, r in zip(got, ref):
        assert_close(g, r, RTOL64, "non-finite inputs")


@pytest.mark.parametrize("name", ["pendulum", "srbm_mpc"])
def test_host_subranges_match_full(name):
    # vsb_eval_host over [e0, e1) of a host workspace (what the INTEGRATION.md run_range stub
    # issues per thread chunk) == the same rows of one full call, bit for bit
    tape = workloads.load_tape(name)
    B = 1000 if name == "pendulum" else 200
    ins = workloads.make_inputs(name, B, seed=31)
    full = gpu_eval(tape, ins)
    ws = BatchWorkspace(tape, B)
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    for o in ws.outputs:
        o[:] = np.nan
    plan = Plan(tape)
    for e0, e1 in [(0, 129), (129, 130), (130, 517), (517, B)] if B == 1000 else [(0, 37), (37, 64), (64, B)]:
        plan.eval_host(ws._in_buf.ctypes.data, ws._in_off, ws._out_buf.ctypes.data, ws._out_off, e0, e1, 0)
    for j in range(tape.n_out):
        assert_bitwise_or_nan(ws.output_matrix(j), full[j], f"{name} out {j}")


@pytest.mark.parametrize("name", ["humanoid_rbd", "srbm_mpc"])
def test_team_kernels_soa_layout_equals_aos(name):
    # team kernels with [nnz, batch] (SoA) I/O (io_ld strides) == the AoS workspace layout, bitwise
    from paper_2408_09662_b200 import Function

    tape = workloads.load_tape(name)
    B = 333
    ins = workloads.make_inputs(name, B, seed=41)
    aos = Function(tape)(*[torch.tensor(v, device="cuda") for v in ins])
    soa = Function(tape, layout="soa")(*[torch.tensor(v.T.copy(), device="cuda") for v in ins])
    for a, s in zip(aos, soa):
        assert_bitwise_or_nan(a.cpu().numpy(), s.cpu().numpy().T, f"{name} soa")


def test_team_kernels_fp32_mode_within_stated_tolerance():
    # fp32 team kernels (humanoid_rbd, team 12): within the stated 1e-4 * max(|ref|, 1)
    from paper_2408_09662_b200 import Function

    tape = workloads.load_tape("humanoid_rbd")
    ins = workloads.make_inputs("humanoid_rbd", 1024, seed=42)
    ref = oracle.batch_eval(tape, ins)
    outs = Function(tape, dtype=torch.float32)(*[torch.tensor(v, dtype=torch.float32, device="cuda") for v in ins])
    for o, r in zip(outs, ref):
        assert_close(o.double().cpu().numpy(), r, RTOL32, "fp32 team")


def test_function_out_argument_is_validated():
    from paper_2408_09662_b200 import Function

    tape = workloads.load_tape("cartpole_rk4")
    ins = [torch.tensor(v, device="cuda") for v in workloads.make_inputs("cartpole_rk4", 64, seed=3)]
    f = Function(tape)
    good = [torch.empty((64, 4), dtype=torch.float64, device="cuda")]
    (o,) = f(*ins, out=good)
    assert o.data_ptr() == good[0].data_ptr()
    bad = [
        [],                                                                        # count
        [torch.empty((63, 4), dtype=torch.float64, device="cuda")],               # shape
        [torch.empty((64, 4), dtype=torch.float32, device="cuda")],               # dtype
        [torch.empty((64, 4), dtype=torch.float64)],                              # device
        [torch.empty((4, 64), dtype=torch.float64, device="cuda").t()],           # layout
    ]
    for out in bad:
        with pytest.raises(ValueError):
            f(*ins, out=out)
    fs = Function(tape, layout="soa")
    sins = [x.t().contiguous() for x in ins]
    wide = torch.empty((4, 80), dtype=torch.float64, device="cuda")[:, :64]      # ld 80 > batch
    (os_,) = fs(*sins, out=[wide])
    assert torch.equal(os_.t(), o)
    with pytest.raises(ValueError):
        fs(*sins, out=[torch.empty((64, 4), dtype=torch.float64, device="cuda")])


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_sharder_over_distinct_devices():
    # vsb_eval_host_sharded over real devices [0, 1, ...]: contiguous B*k//W shards
    # (batchrt.py:189-191), one host thread + stream set per GPU, no collective
    n = min(torch.cuda.device_count(), 8)
    tape = workloads.load_tape("srbm_mpc")
    B = 1000 + n * 37
    ins = workloads.make_inputs("srbm_mpc", B, seed=88)
    ws = BatchWorkspace(tape, B)
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    batch_eval(tape, ws, devices=list(range(n)))
    ref = oracle.batch_eval(tape, ins, n_threads=8)
    for j, r in enumerate(ref):
        assert_close(ws.output_matrix(j), r, RTOL64, f"sharded over {n} GPUs out {j}")
    assert torch.cuda.current_device() == 0   # the device guard restored the caller's device


def test_value_numbering_is_bitwise_on_special_values():
    # the merged rows and identities hold for every IEEE class (signed zeros, subnormals,
    # infinities, NaN): GPU == oracle (the reference's run_range restated) bit for bit
    from vn_tapes import vn_inputs, vn_tape

    tape, ins = vn_tape(), vn_inputs()
    ref = oracle.batch_eval(tape, ins)
    got = gpu_eval(tape, ins)
    assert_bitwise_or_nan(got[0], ref[0], "value numbering")
