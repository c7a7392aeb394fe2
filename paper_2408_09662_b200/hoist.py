"""Loop-invariant hoisting for closed-loop rollouts.

A rollout evaluates ``state_{k+1} = f(state_k, params)`` K times
(``quadsim.rollout_batch`` / ``roa_scan``, /root/reference/pkg/src/vecsym/
quadsim.py:298-303,367-369).  Most of such a tape often depends on the
parameters alone -- quad_step's in-graph LQR synthesis (quadsim.py:216-222)
is 42,501 of its 42,553 arithmetic rows; only 52 touch the state.
``split_invariant`` cuts a tape into

* ``pre``  (parameter inputs -> one dense "boundary" output): every row that
  does not depend on a varying input, with an OUTPUT row for each of its
  values the varying part consumes, and
* ``step`` (varying inputs + the boundary -> the original outputs): the rows
  that do depend on a varying input, reading invariant operands from the
  boundary input (CONST operands are re-emitted as CONST rows).

Every row of the original tape is evaluated by exactly one of the two, on the
same operand values, so ``step(varying, pre(params))`` is bit for bit
``f(varying, params)``.  The tapes use the reference's row format (tape.py:
10-20) and pass its validation (tape.py:171-258).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tape import ARITY, InstructionTape, OpCode, as_tape

__all__ = ["InvariantSplit", "split_invariant"]

_INPUT, _OUTPUT, _CONST = int(OpCode.INPUT), int(OpCode.OUTPUT), int(OpCode.CONST)


@dataclass(frozen=True)
class InvariantSplit:
    pre: InstructionTape          # inputs: the non-varying inputs in order; output 0: boundary [m]
    step: InstructionTape         # inputs: the varying inputs in order, then the boundary; outputs: original
    varying: tuple                # original indices of the varying inputs
    fixed: tuple                  # original indices of the other inputs (the pre tape's inputs)
    hoisted_rows: int             # arithmetic rows moved to the pre tape
    step_rows: int                # arithmetic rows left in the step tape

    @property
    def boundary(self) -> int:
        return self.pre.nnz_out[0]


def split_invariant(tape, varying=(0,)):
    """Split ``tape`` into invariant/varying parts (see module doc).

    Returns None when nothing would be hoisted (no arithmetic row is
    independent of the varying inputs, or the step tape would need no
    boundary value).
    """
    t = as_tape(tape)
    code, values = t.packed()
    varying = tuple(sorted({int(v) for v in varying}))
    if any(v < 0 or v >= t.n_in for v in varying):
        raise ValueError(f"varying inputs {varying} out of range for {t.n_in} inputs")
    fixed = tuple(i for i in range(t.n_in) if i not in varying)
    n = code.shape[0]
    ops = code[:, 0].tolist()
    rows = code.tolist()

    # SSA pass: the value a row defines is named by the row index
    slot_val = {}
    tainted = bytearray(n)
    operands = [()] * n
    is_var = set(varying)
    for i, (op, out, a, b, c) in enumerate(rows):
        if op == _INPUT:
            tainted[i] = a in is_var
            slot_val[out] = i
        elif op == _CONST:
            slot_val[out] = i
        elif op == _OUTPUT:
            operands[i] = (slot_val[a],)
        else:
            vs = tuple(slot_val[s] for s in (a, b, c)[:ARITY[op]])
            operands[i] = vs
            tainted[i] = any(tainted[v] for v in vs)
            slot_val[out] = i

    # boundary: invariant, non-constant values read by the step part
    need = set()
    consts = set()
    for i in range(n):
        if tainted[i] or ops[i] == _OUTPUT:
            for v in operands[i]:
                if tainted[v]:
                    continue
                (consts if ops[v] == _CONST else need).add(v)
    boundary = sorted(need)
    plumbing = {_INPUT, _OUTPUT, _CONST, int(OpCode.ASSIGN)}
    hoisted = sum(1 for i in range(n) if not tainted[i] and ops[i] not in plumbing)
    step_rows = sum(1 for i in range(n) if tainted[i] and ops[i] not in plumbing)
    if hoisted == 0 or not boundary:
        return None
    bpos = {v: k for k, v in enumerate(boundary)}

    # pre tape: invariant rows in order, each boundary value stored right after its row
    fmap = {old: k for k, old in enumerate(fixed)}
    pre_code, pre_vals = [], []
    for i, (op, out, a, b, c) in enumerate(rows):
        if tainted[i] or op == _OUTPUT:
            continue
        pre_code.append([op, out, fmap[a], b, c] if op == _INPUT else [op, out, a, b, c])
        pre_vals.append(values[i])
        if i in bpos:
            pre_code.append([_OUTPUT, 0, out, bpos[i], -1])
            pre_vals.append(0.0)
    pre = InstructionTape(f"{t.name}_pre", np.asarray(pre_code, dtype=np.int32).reshape(-1, 5), pre_vals, t.n_w,
                          [t.input_sparsity[i] for i in fixed], [len(boundary)])

    # step tape: SSA slots; boundary INPUT rows first, then constants / varying rows / stores
    vmap = {old: k for k, old in enumerate(varying)}
    nb = len(varying)
    new_slot = {}
    st_code, st_vals = [], []

    def define(v, row, val=0.0):
        new_slot[v] = len(new_slot)
        row[1] = new_slot[v]
        st_code.append(row)
        st_vals.append(val)

    for v in boundary:
        define(v, [_INPUT, 0, nb, bpos[v], -1])
    for i, (op, out, a, b, c) in enumerate(rows):
        if op == _OUTPUT:
            st_code.append([_OUTPUT, out, new_slot[operands[i][0]], b, -1])
            st_vals.append(0.0)
        elif op == _CONST:
            if i in consts:
                define(i, [_CONST, 0, -1, -1, -1], values[i])
        elif tainted[i]:
            if op == _INPUT:
                define(i, [_INPUT, 0, vmap[a], b, -1])
            else:
                args = [new_slot[v] for v in operands[i]] + [-1] * (3 - len(operands[i]))
                define(i, [op, 0] + args)
    step = InstructionTape(f"{t.name}_step", np.asarray(st_code, dtype=np.int32).reshape(-1, 5), st_vals,
                           max(1, len(new_slot)),
                           [t.input_sparsity[i] for i in varying] + [len(boundary)], list(t.output_sparsity))
    return InvariantSplit(pre, step, varying, fixed, hoisted, step_rows)
