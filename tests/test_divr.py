"""Shared-reciprocal division (codegen DIVR: one RN(1/b) per divisor + FMA
corrections, IEEE fallback outside 2^+-250) must be bit-identical to IEEE
division on every input class: random bit patterns over the whole double
range (subnormals, zeros, infinities, NaNs), all-ones significands,
quotients at the fallback boundaries."""

import numpy as np
import pytest

import oracle
from paper_2408_09662_b200.tape import InstructionTape, OpCode

from conftest import assert_bitwise_or_nan

K = 8


def divr_tape():
    # inputs: a[K], b[1]; outputs: a_k / b (shared divisor), a_k / 3.0 (shared constant), b / a_0
    rows, vals = [], []
    for k in range(K):
        rows.append([int(OpCode.INPUT), k, 0, k, -1]); vals.append(0.0)
    rows.append([int(OpCode.INPUT), K, 1, 0, -1]); vals.append(0.0)
    rows.append([int(OpCode.CONST), K + 1, -1, -1, -1]); vals.append(3.0)
    slot = K + 2
    for k in range(K):
        rows.append([int(OpCode.DIV), slot, k, K, -1]); vals.append(0.0)
        rows.append([int(OpCode.OUTPUT), 0, slot, k, -1]); vals.append(0.0)
        rows.append([int(OpCode.DIV), slot + 1, k, K + 1, -1]); vals.append(0.0)
        rows.append([int(OpCode.OUTPUT), 1, slot + 1, k, -1]); vals.append(0.0)
    rows.append([int(OpCode.DIV), slot, K, 0, -1]); vals.append(0.0)
    rows.append([int(OpCode.OUTPUT), 2, slot, 0, -1]); vals.append(0.0)
    return InstructionTape("divr", np.array(rows, dtype=np.int32), vals, slot + 2, [K, 1], [K, K, 1])


def divr_inputs(B, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2**64, size=(B, K + 1), dtype=np.uint64, endpoint=False)
    x = bits.view(np.float64).copy()
    n = B // 4
    # moderate exponents (the DIVR fast path) for half the rows
    x[n:2 * n] = rng.normal(size=(n, K + 1)) * np.exp2(rng.integers(-300, 300, size=(n, K + 1)))
    x[2 * n:3 * n] = rng.normal(size=(n, K + 1))
    # all-ones significands, powers of two, boundary exponents
    m = x[3 * n:]
    m[:, :] = np.exp2(rng.integers(-260, 260, size=m.shape).astype(float))
    ones = rng.random(m.shape) < 0.5
    m[ones] *= (2.0 - 2.0**-52)
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 2.0**-1022, 2.0**-250, 2.0**250,
                         2.0**-251, 2.0**251, 1.0, -1.0, 3.0, 1.0 / 3.0])
    sel = rng.random(x.shape) < 0.03
    x[sel] = rng.choice(specials, size=int(sel.sum()))
    return [x[:, :K].copy(), x[:, K:].copy()]


def test_divr_oracle_matches_numpy():
    # the oracle's DIV is IEEE division (numpy divide, same bits)
    t = divr_tape()
    ins = divr_inputs(4096, 1)
    outs = oracle.batch_eval(t, ins)
    with np.errstate(all="ignore"):
        assert_bitwise_or_nan(outs[0], ins[0] / ins[1], "a/b")
        assert_bitwise_or_nan(outs[1], ins[0] / 3.0, "a/3")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [2, 3])
def test_divr_bitwise_vs_ieee_division(seed, monkeypatch):
    import paper_2408_09662_b200 as vsb

    monkeypatch.setenv("VSB_DIV_RECIP", "1")   # opt-in codegen path
    vsb.clear_plan_cache()
    t = divr_tape()
    B = 1 << 20
    ins = divr_inputs(B, seed)
    ref = oracle.batch_eval(t, ins, n_threads=8)
    ws = vsb.BatchWorkspace(t, B)
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    vsb.batch_eval(t, ws)
    for j in range(3):
        assert_bitwise_or_nan(ws.output_matrix(j), ref[j], f"out {j}")
    src = vsb.get_plan(t).source(0)
    assert "vs_divr(" in src and "vs_rcp_o(" in src
    vsb.clear_plan_cache()
