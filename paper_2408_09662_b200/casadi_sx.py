"""Ingest a casadi SX ``Function`` (or its instruction list) as an instruction tape.

``north_star`` asks the evaluator to "load a casadi Function or its serialized
SX instruction tape".  casadi is not a dependency of the reference
(/root/reference/pkg has no casadi import) and is not installed
in this image, so this adapter is **parity unpinned**: it follows casadi's
published SX algorithm semantics (one ``ScalarAtomic`` per instruction:
``OP_CONST w[i0] = d``, ``OP_INPUT w[i0] = in[i1][i2]``, ``OP_OUTPUT
out[i0][i2] = w[i1]``, unary/binary ``w[i0] = f(w[i1][, w[i2]])``) and reads
the opcodes by *name* from the installed ``casadi`` module (``casadi.OP_ADD``
...), never from hard-coded numbers.

Two entry points:

* :func:`from_casadi` walks a live ``casadi.Function`` through its public
  instruction API (``n_instructions``, ``instruction_id``,
  ``instruction_input``, ``instruction_output``, ``instruction_constant``,
  ``sparsity_in/out``, ``sz_w``).
* :func:`from_instructions` takes the same information as plain data
  (opcode names, work/IO indices, constants): the form a serialized SX tape
  reduces to, and what the tests drive.

casadi ops without a counterpart in the tape IR are lowered exactly where an
exact rewrite exists (``OP_TWICE x`` -> ``x + x``, ``OP_INV x`` -> ``1 / x``,
``OP_CONSTPOW`` -> ``POW``, ``OP_IF_ELSE_ZERO c x`` -> ``IF_ELSE(c, x, 0)``)
and rejected otherwise with the instruction index in the message (the
reference's ``"instruction i: ..."`` wording, tape.py:73-77).
"""

from __future__ import annotations

from typing import Iterable, Sequence

import numpy as np

from .tape import InstructionTape, OpCode, Sparsity, TapeError

__all__ = ["from_casadi", "from_instructions", "SUPPORTED_OPS"]

# casadi op name -> (tape opcode, arity); exact one-to-one maps
_DIRECT = {
    "OP_ASSIGN": (OpCode.ASSIGN, 1), "OP_ADD": (OpCode.ADD, 2), "OP_SUB": (OpCode.SUB, 2),
    "OP_MUL": (OpCode.MUL, 2), "OP_DIV": (OpCode.DIV, 2), "OP_NEG": (OpCode.NEG, 1),
    "OP_EXP": (OpCode.EXP, 1), "OP_LOG": (OpCode.LOG, 1), "OP_POW": (OpCode.POW, 2),
    "OP_CONSTPOW": (OpCode.POW, 2), "OP_SQRT": (OpCode.SQRT, 1), "OP_SQ": (OpCode.SQ, 1),
    "OP_SIN": (OpCode.SIN, 1), "OP_COS": (OpCode.COS, 1), "OP_TAN": (OpCode.TAN, 1),
    "OP_ATAN2": (OpCode.ATAN2, 2), "OP_FABS": (OpCode.FABS, 1), "OP_FMIN": (OpCode.FMIN, 2),
    "OP_FMAX": (OpCode.FMAX, 2),
}
# exact lowerings onto IR sequences (comparisons and logic yield 1.0 / 0.0 like casadi's
# casadi_math: x < y, x <= y, x == y, x != y, !x, x && y, x || y; NaN is truthy)
_LOWERED = ("OP_TWICE", "OP_INV", "OP_IF_ELSE_ZERO", "OP_LT", "OP_LE", "OP_EQ", "OP_NE", "OP_NOT", "OP_AND",
            "OP_OR")
_PLUMBING = ("OP_CONST", "OP_INPUT", "OP_OUTPUT")
SUPPORTED_OPS = tuple(_DIRECT) + _LOWERED + _PLUMBING


def _lt(emit, o, x, y, t):
    """o = (x < y) = STEP(y - x): y - x > 0 exactly when y > x for every IEEE pair (gradual
    underflow keeps a nonzero difference nonzero, overflow keeps its sign; inf - inf and
    NaN give NaN, and STEP(NaN) = 0 = (x < y))."""
    emit(OpCode.SUB, t, y, x)
    emit(OpCode.STEP, o, t)


def _not(emit, o, x, t):
    """o = !x = (x == 0): IF_ELSE(x, 0, 1) (NaN != 0 is truthy, as in C)."""
    emit(OpCode.CONST, t, v=0.0)
    emit(OpCode.CONST, t + 1, v=1.0)
    emit(OpCode.IF_ELSE, o, x, t, t + 1)


def _le(emit, o, x, y, t):
    """o = (x <= y) = !(y < x) * ordered(x, y); ordered(v) = STEP(|v| + 1) (0 only for NaN).
    inf <= inf: y < x is STEP(inf - inf) = 0, so the result is 1 as it must be."""
    _lt(emit, t, y, x, t + 1)              # t = y < x
    _not(emit, t, t, t + 1)                # t = !(y < x)
    emit(OpCode.CONST, t + 1, v=1.0)
    for v in (x, y):
        emit(OpCode.FABS, t + 2, v)
        emit(OpCode.ADD, t + 2, t + 2, t + 1)
        emit(OpCode.STEP, t + 2, t + 2)    # 1 unless v is NaN
        emit(OpCode.MUL, t, t, t + 2)
    emit(OpCode.ASSIGN, o, t)


def _lower_lt(emit, o, a, t):
    _lt(emit, t, a[0], a[1], t + 1)
    emit(OpCode.ASSIGN, o, t)
    return 2


def _lower_le(emit, o, a, t):
    _le(emit, o, a[0], a[1], t)
    return 3


def _lower_eq(emit, o, a, t):
    # x == y  <=>  x <= y and y <= x (both 0/1: the product is exact); NaN: 0
    _le(emit, t + 3, a[0], a[1], t)
    _le(emit, t + 4, a[1], a[0], t)
    emit(OpCode.MUL, o, t + 3, t + 4)
    return 5


def _lower_ne(emit, o, a, t):
    _lower_eq(emit, t + 5, a, t)
    _not(emit, o, t + 5, t)
    return 6


def _lower_not(emit, o, a, t):
    _not(emit, t + 2, a[0], t)
    emit(OpCode.ASSIGN, o, t + 2)
    return 3


def _lower_and(emit, o, a, t):
    # x && y: IF_ELSE(x, IF_ELSE(y, 1, 0), 0)
    emit(OpCode.CONST, t, v=0.0)
    emit(OpCode.CONST, t + 1, v=1.0)
    emit(OpCode.IF_ELSE, t + 2, a[1], t + 1, t)
    emit(OpCode.IF_ELSE, o, a[0], t + 2, t)
    return 3


def _lower_or(emit, o, a, t):
    # x || y: IF_ELSE(x, 1, IF_ELSE(y, 1, 0))
    emit(OpCode.CONST, t, v=0.0)
    emit(OpCode.CONST, t + 1, v=1.0)
    emit(OpCode.IF_ELSE, t + 2, a[1], t + 1, t)
    emit(OpCode.IF_ELSE, o, a[0], t + 1, t + 2)
    return 3


# op name -> lowering(emit, out slot, operand slots, first scratch slot) -> scratch slots used;
# every lowering reads its operands before it writes `out` (casadi may reuse an operand slot)
_LOGIC = {"OP_LT": _lower_lt, "OP_LE": _lower_le, "OP_EQ": _lower_eq, "OP_NE": _lower_ne, "OP_NOT": _lower_not,
          "OP_AND": _lower_and, "OP_OR": _lower_or}


def _sparsity(sp) -> Sparsity:
    """casadi Sparsity (size1/size2/colind/row) or ours or an int."""
    if isinstance(sp, (Sparsity, int, np.integer)):
        return sp if isinstance(sp, Sparsity) else Sparsity.dense(int(sp), 1)
    return Sparsity(sp.size1(), sp.size2(), list(sp.colind()), list(sp.row()))


def from_instructions(name: str, instructions: Iterable[Sequence], n_w: int, input_sparsity, output_sparsity,
                      ) -> InstructionTape:
    """Build a tape from casadi-style instructions.

    Each instruction is ``(op_name, outputs, inputs, constant)`` exactly as
    casadi's ``instruction_output(k)`` / ``instruction_input(k)`` /
    ``instruction_constant(k)`` report them:

    * ``OP_CONST``: outputs ``[i0]``, constant ``d``
    * ``OP_INPUT``: outputs ``[i0]``, inputs ``[input index, nonzero]``
    * ``OP_OUTPUT``: outputs ``[output index, nonzero]``, inputs ``[i1]``
    * others: outputs ``[i0]``, inputs = work operands
    """
    ins_sp = [_sparsity(s) for s in input_sparsity]
    outs_sp = [_sparsity(s) for s in output_sparsity]
    rows: list[tuple[int, int, int, int, int]] = []
    vals: list[float] = []
    scratch = int(n_w)  # extra work slots for lowerings (allocated past casadi's sz_w)
    extra = 0

    def emit(op, o, a=-1, b=-1, c=-1, v=0.0):  # -1 sentinels in unused fields (tape.py validation)
        rows.append((int(op), int(o), int(a), int(b), int(c)))
        vals.append(float(v))

    for k, ins in enumerate(instructions):
        op_name, outs, args, const = ins
        outs = [int(x) for x in outs]
        args = [int(x) for x in args]
        try:
            if op_name == "OP_CONST":
                emit(OpCode.CONST, outs[0], v=const)
            elif op_name == "OP_INPUT":
                emit(OpCode.INPUT, outs[0], args[0], args[1])
            elif op_name == "OP_OUTPUT":
                emit(OpCode.OUTPUT, outs[0], args[0], outs[1])
            elif op_name in _DIRECT:
                op, ar = _DIRECT[op_name]
                if len(args) < ar:
                    raise TapeError(f"instruction {k}: {op_name} needs {ar} operands, got {len(args)}")
                emit(op, outs[0], *args[:ar])
            elif op_name == "OP_TWICE":
                emit(OpCode.ADD, outs[0], args[0], args[0])
            elif op_name == "OP_INV":
                one = scratch
                extra = max(extra, 1)
                emit(OpCode.CONST, one, v=1.0)
                emit(OpCode.DIV, outs[0], one, args[0])
            elif op_name == "OP_IF_ELSE_ZERO":
                zero = scratch
                extra = max(extra, 1)
                emit(OpCode.CONST, zero, v=0.0)
                emit(OpCode.IF_ELSE, outs[0], args[0], args[1], zero)
            elif op_name in _LOGIC:
                extra = max(extra, _LOGIC[op_name](emit, outs[0], args, scratch))
            else:
                raise TapeError(f"instruction {k}: casadi operation {op_name} has no tape equivalent "
                                f"(supported: {', '.join(SUPPORTED_OPS)})")
        except IndexError:
            raise TapeError(f"instruction {k}: malformed {op_name} (outputs {outs}, inputs {args})") from None
    code = np.asarray(rows, dtype=np.int32).reshape(-1, 5)
    return InstructionTape(name, code, np.asarray(vals, dtype=np.float64), int(n_w) + extra, ins_sp, outs_sp)


def _op_names(casadi_module) -> dict:
    """opcode number -> name, read from the installed casadi module."""
    names = {}
    for attr in dir(casadi_module):
        if attr.startswith("OP_"):
            val = getattr(casadi_module, attr)
            if isinstance(val, (int, np.integer)):
                names.setdefault(int(val), attr)
    return names


def from_casadi(f, *, casadi_module=None, name: str | None = None) -> InstructionTape:
    """Tape of an SX ``casadi.Function`` (parity unpinned: casadi is absent here)."""
    if casadi_module is None:
        try:
            import casadi as casadi_module  # noqa: F401
        except ImportError as exc:
            raise ImportError("from_casadi needs the casadi package (not installed); "
                              "use from_instructions for a serialized instruction list") from exc
    if hasattr(f, "is_a") and not f.is_a("SXFunction"):
        raise ValueError(f"function {f.name()!r} is not an SX function (expand it first: f.expand())")
    names = _op_names(casadi_module)

    def gen():
        for k in range(f.n_instructions()):
            op = int(f.instruction_id(k))
            if op not in names:
                raise TapeError(f"instruction {k}: unknown casadi opcode {op}")
            nm = names[op]
            const = f.instruction_constant(k) if nm == "OP_CONST" else 0.0
            yield nm, list(f.instruction_output(k)), list(f.instruction_input(k)), const

    nm = name or f.name()
    if not str(nm).isidentifier():
        nm = "casadi_" + "".join(ch if ch.isalnum() else "_" for ch in str(nm))
    return from_instructions(nm, gen(), int(f.sz_w()), [f.sparsity_in(i) for i in range(f.n_in())],
                             [f.sparsity_out(j) for j in range(f.n_out())])
