"""casadi SX ingest (``paper_2408_09662_b200.casadi_sx``) -- parity UNPINNED.

casadi is neither a reference dependency nor installed, so
these tests drive the adapter with a stand-in ``casadi`` module whose OP_*
numbers deliberately differ from the tape IR's (the adapter must map by
name) and a stand-in ``Function`` exposing casadi's instruction API for
f(x, y) = [sin(x0)*y + 2*x1 (OP_TWICE), if_else_zero(x0, 1/y) (OP_INV)].
The resulting tape is checked against numpy on CPU (oracle) and on the GPU.
"""

import types

import numpy as np
import pytest

from paper_2408_09662_b200.casadi_sx import SUPPORTED_OPS, from_casadi, from_instructions
from paper_2408_09662_b200.tape import TapeError, deserialize, serialize

_NAMES = ["OP_ASSIGN", "OP_ADD", "OP_SUB", "OP_MUL", "OP_DIV", "OP_NEG", "OP_EXP", "OP_LOG", "OP_POW",
          "OP_CONSTPOW", "OP_SQRT", "OP_SQ", "OP_TWICE", "OP_SIN", "OP_COS", "OP_TAN", "OP_LT", "OP_FABS",
          "OP_IF_ELSE_ZERO", "OP_FMIN", "OP_FMAX", "OP_INV", "OP_ATAN2", "OP_CONST", "OP_INPUT", "OP_OUTPUT",
          "OP_FLOOR"]
FAKE_CASADI = types.SimpleNamespace(**{n: 100 + 7 * i for i, n in enumerate(_NAMES)})


class FakeSparsity:
    def __init__(self, n):
        self.n = n

    def size1(self):
        return self.n

    def size2(self):
        return 1

    def colind(self):
        return [0, self.n]

    def row(self):
        return list(range(self.n))


class FakeFunction:
    """casadi.Function-like: instructions are (name, outputs, inputs, const)."""

    def __init__(self, instr, sz_w, n_in, n_out, name="f"):
        self.instr, self._sz_w, self._in, self._out, self._name = instr, sz_w, n_in, n_out, name

    def is_a(self, kind):
        return kind == "SXFunction"

    def name(self):
        return self._name

    def n_instructions(self):
        return len(self.instr)

    def instruction_id(self, k):
        return getattr(FAKE_CASADI, self.instr[k][0])

    def instruction_output(self, k):
        return self.instr[k][1]

    def instruction_input(self, k):
        return self.instr[k][2]

    def instruction_constant(self, k):
        return self.instr[k][3]

    def sz_w(self):
        return self._sz_w

    def n_in(self):
        return len(self._in)

    def n_out(self):
        return len(self._out)

    def sparsity_in(self, i):
        return FakeSparsity(self._in[i])

    def sparsity_out(self, j):
        return FakeSparsity(self._out[j])


# x: input 0 (2 nz), y: input 1 (1 nz); out0 = sin(x0)*y + twice(x1); out1 = if_else_zero(x0, inv(y))
INSTR = [
    ("OP_INPUT", [0], [0, 0], 0.0),
    ("OP_INPUT", [1], [0, 1], 0.0),
    ("OP_INPUT", [2], [1, 0], 0.0),
    ("OP_SIN", [3], [0], 0.0),
    ("OP_MUL", [3], [3, 2], 0.0),
    ("OP_TWICE", [1], [1], 0.0),
    ("OP_ADD", [3], [3, 1], 0.0),
    ("OP_OUTPUT", [0, 0], [3], 0.0),
    ("OP_INV", [2], [2], 0.0),
    ("OP_IF_ELSE_ZERO", [2], [0, 2], 0.0),
    ("OP_CONST", [1], [], 0.25),
    ("OP_MUL", [2], [2, 1], 0.0),
    ("OP_OUTPUT", [1, 0], [2], 0.0),
]


def expected(x, y):
    o0 = np.sin(x[:, 0]) * y[:, 0] + (x[:, 1] + x[:, 1])
    o1 = np.where(x[:, 0] != 0, 1.0 / y[:, 0], 0.0) * 0.25
    return o0[:, None], o1[:, None]


def make_inputs(n=64):
    rng = np.random.default_rng(7)
    x = rng.uniform(-2, 2, size=(n, 2))
    x[::5, 0] = 0.0                     # exercise the if_else_zero false branch
    y = rng.uniform(0.5, 3, size=(n, 1))
    return x, y


def test_from_casadi_maps_opcodes_by_name():
    tape = from_casadi(FakeFunction(INSTR, 4, [2, 1], [1, 1]), casadi_module=FAKE_CASADI)
    assert tape.nnz_in == [2, 1] and tape.nnz_out == [1, 1]
    assert tape.n_w == 5                      # casadi's sz_w + one lowering temp
    text = serialize(tape)
    assert deserialize(text).digest() == tape.digest()   # round-trips through the v1 format


def test_from_casadi_values_match_numpy_on_cpu_oracle():
    import oracle

    tape = from_casadi(FakeFunction(INSTR, 4, [2, 1], [1, 1]), casadi_module=FAKE_CASADI)
    x, y = make_inputs()
    got = oracle.batch_eval(tape, [x, y])
    for g, e in zip(got, expected(x, y)):
        np.testing.assert_array_equal(g, e)   # sin via glibc on both sides


def test_unsupported_op_names_instruction():
    bad = INSTR[:3] + [("OP_FLOOR", [3], [0], 0.0)] + INSTR[3:]
    with pytest.raises(TapeError, match="instruction 3: casadi operation OP_FLOOR"):
        from_casadi(FakeFunction(bad, 4, [2, 1], [1, 1]), casadi_module=FAKE_CASADI)


def test_unknown_opcode_and_non_sx_rejected():
    f = FakeFunction(INSTR, 4, [2, 1], [1, 1])
    f.instruction_id = lambda k: 99999
    with pytest.raises(TapeError, match="unknown casadi opcode"):
        from_casadi(f, casadi_module=FAKE_CASADI)
    g = FakeFunction(INSTR, 4, [2, 1], [1, 1])
    g.is_a = lambda kind: False
    with pytest.raises(ValueError, match="not an SX function"):
        from_casadi(g, casadi_module=FAKE_CASADI)


def test_from_instructions_validates_like_the_tape():
    # read before write is caught by the tape validator with the row index
    with pytest.raises(TapeError, match="instruction 0"):
        from_instructions("g", [("OP_ADD", [0], [1, 2], 0.0)], 3, [1], [1])
    assert "OP_IF_ELSE_ZERO" in SUPPORTED_OPS


def test_missing_casadi_is_a_clear_import_error():
    try:
        import casadi  # noqa: F401
        pytest.skip("casadi installed")
    except ImportError:
        pass
    with pytest.raises(ImportError, match="from_instructions"):
        from_casadi(FakeFunction(INSTR, 4, [2, 1], [1, 1]))


@pytest.mark.gpu
def test_casadi_tape_on_gpu():
    import paper_2408_09662_b200 as vsb
    from conftest import assert_close

    tape = from_casadi(FakeFunction(INSTR, 4, [2, 1], [1, 1]), casadi_module=FAKE_CASADI)
    x, y = make_inputs(1000)
    ws = vsb.BatchWorkspace(tape, x.shape[0])
    ws.set_input(0, x)
    ws.set_input(1, y)
    vsb.batch_eval(tape, ws)
    for j, e in enumerate(expected(x, y)):
        assert_close(ws.output_matrix(j), e)


_SPECIAL = np.array([0.0, -0.0, 1.0, -1.0, 2.5, -2.5, 1e-310, -1e-310, 5e-324, 1e308, -1e308, np.inf, -np.inf, np.nan])
_CMP = {
    "OP_LT": lambda x, y: x < y, "OP_LE": lambda x, y: x <= y, "OP_EQ": lambda x, y: x == y,
    "OP_NE": lambda x, y: x != y, "OP_AND": lambda x, y: (x != 0) & (y != 0), "OP_OR": lambda x, y: (x != 0) | (y != 0),
    "OP_NOT": lambda x, y: x == 0,
}


@pytest.mark.parametrize("op", sorted(_CMP))
@pytest.mark.parametrize("alias", [False, True])
def test_comparison_and_logic_lowerings_exact(op, alias):
    """casadi's comparison / logic ops (1.0 or 0.0, NaN truthy, IEEE ordering incl. signed zeros,
    infinities, subnormals and NaN) lowered onto STEP / IF_ELSE / FABS / arithmetic rows:
    checked against numpy's comparisons on every pair of special values (CPU oracle).
    ``alias``: the result overwrites an operand's work slot, as casadi's register reuse does."""
    import oracle

    x = np.repeat(_SPECIAL, _SPECIAL.size)[:, None]
    y = np.tile(_SPECIAL, _SPECIAL.size)[:, None]
    out = 0 if alias else 2
    args = [0] if op == "OP_NOT" else [0, 1]
    instr = [("OP_INPUT", [0], [0, 0], 0.0), ("OP_INPUT", [1], [1, 0], 0.0), (op, [out], args, 0.0),
             ("OP_OUTPUT", [0, 0], [out], 0.0)]
    tape = from_instructions("cmp", instr, 3, [1, 1], [1])
    (got,) = oracle.batch_eval(tape, [x, y])
    want = _CMP[op](x, y).astype(np.float64)
    bad = np.flatnonzero(got[:, 0] != want[:, 0])
    assert bad.size == 0, [(x[i, 0], y[i, 0], got[i, 0], want[i, 0]) for i in bad[:5]]
    assert not np.signbit(got).any()
