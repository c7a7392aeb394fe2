"""Explain a GPU-vs-reference difference by libm rounding alone (test infrastructure).

For a row whose GPU output disagrees with the reference beyond what the 1-ulp sensitivity
patterns predict (a kink flipped by the particular ulps another libm returns), this module

1. traces the GPU value of every arithmetic row for that row (the tape instrumented with one
   extra output per arithmetic row, evaluated through the C ABI),
2. replays the tape in IEEE double on the CPU with the reference's op semantics
   (oracle/vs_oracle.c, i.e. _kernels.py:54-206), taking every transcendental result
   (exp, log, pow, sin, cos, tan, atan2) from the GPU trace and computing everything else,
3. accepts the row iff the replay reproduces the GPU outputs bit for bit (NaN == NaN) and
   every substituted transcendental is within ``max_ulps`` of the glibc value for the same
   operands.

Acceptance therefore proves: the GPU result is the exact evaluation of the tape under a libm
whose every result lies within ``max_ulps`` of glibc's -- a conforming libm (libdevice
documents <= 2 ulp for pow / tan / atan2, <= 1 for exp / log; sin / cos here are correctly
rounded).
"""

from __future__ import annotations

import math

import numpy as np

from paper_2408_09662_b200 import BatchWorkspace, InstructionTape, batch_eval

CONST, INPUT, OUTPUT, ASSIGN = 0, 1, 2, 3
ADD, SUB, MUL, DIV, NEG, EXP, LOG, POW, SQRT, SQ, SIN, COS, TAN, ATAN2, FABS, FMIN, FMAX, STEP, IF_ELSE = range(4, 23)
TRANSCENDENTAL = {EXP, LOG, POW, SIN, COS, TAN, ATAN2}


def gpu_trace(tape, inputs, plan_options=None):
    """GPU value of every arithmetic row, [rows, n_arith], plus the arithmetic row indices."""
    code, vals = tape.packed()
    arith = [r for r in range(code.shape[0]) if code[r, 0] > ASSIGN]
    pos = {r: k for k, r in enumerate(arith)}
    extra = len(tape.nnz_out)
    rows, values = [], []
    for r in range(code.shape[0]):
        rows.append(code[r].tolist())
        values.append(vals[r])
        if code[r, 0] > ASSIGN:
            rows.append([OUTPUT, extra, int(code[r, 1]), pos[r], -1])
            values.append(0.0)
    traced = InstructionTape(tape.name + "_traced", np.array(rows, dtype=np.int32), np.array(values), tape.n_w,
                             list(tape.nnz_in), list(tape.nnz_out) + [len(arith)])
    ws = BatchWorkspace(traced, inputs[0].shape[0])
    for i, v in enumerate(inputs):
        ws.set_input(i, v)
    batch_eval(traced, ws, plan_options=plan_options)
    return ws.output_matrix(extra).copy(), arith


def _glibc(op, x, y):
    """glibc's value for the same operands (Python's math module), numpy for the special cases
    math signals with exceptions (overflow, domain errors)."""
    f = {EXP: math.exp, LOG: math.log, SIN: math.sin, COS: math.cos, TAN: math.tan}
    try:
        if op in f:
            return f[op](x)
        if op == POW:
            return math.pow(x, y)
        if op == ATAN2:
            return math.atan2(x, y)
    except (OverflowError, ValueError):
        pass
    x, y = np.float64(x), np.float64(y)
    with np.errstate(all="ignore"):
        if op == LOG:
            return float(np.log(x)) if x >= 0 or x != x else math.nan
        g = {EXP: np.exp, SIN: np.sin, COS: np.cos, TAN: np.tan}.get(op)
        if g is not None:
            return float(g(x))
        if op == POW:
            return float(np.power(x, y))
        if op == ATAN2:
            return float(np.arctan2(x, y))
    raise ValueError(op)


def _ulps(a, b):
    if math.isnan(a) and math.isnan(b):
        return 0
    if math.isnan(a) or math.isnan(b):
        return math.inf
    if a == b:
        return 0
    ia = int(np.float64(a).view(np.int64))
    ib = int(np.float64(b).view(np.int64))
    if (ia < 0) != (ib < 0):   # different signs: distance through zero
        return abs(ia & 0x7FFFFFFFFFFFFFFF) + abs(ib & 0x7FFFFFFFFFFFFFFF)
    return abs(ia - ib)


def replay_row(tape, row_inputs, trace_row, arith):
    """CPU replay of one row with the transcendental results taken from the GPU trace.
    Returns (outputs: list of arrays, worst ulp distance of a substituted result to glibc)."""
    code, vals = tape.packed()
    pos = {r: k for k, r in enumerate(arith)}
    w = [0.0] * max(tape.n_w, 1)
    outs = [np.zeros(n) for n in tape.nnz_out]
    worst = 0
    for r in range(code.shape[0]):
        op, o, a, b, c = (int(v) for v in code[r])
        if op == CONST:
            w[o] = float(vals[r])
        elif op == INPUT:
            w[o] = float(row_inputs[a][b])
        elif op == OUTPUT:
            outs[o][b] = w[a]
        elif op == ASSIGN:
            w[o] = w[a]
        elif op in TRANSCENDENTAL:
            g = float(trace_row[pos[r]])
            ref = _glibc(op, w[a], w[b] if op in (POW, ATAN2) else 0.0)
            worst = max(worst, _ulps(g, ref))
            w[o] = g
        else:
            x = np.float64(w[a])
            y = np.float64(w[b]) if b >= 0 else np.float64(0.0)
            with np.errstate(all="ignore"):
                if op == ADD:
                    v = x + y
                elif op == SUB:
                    v = x - y
                elif op == MUL:
                    v = x * y
                elif op == DIV:
                    v = x / y
                elif op == NEG:
                    v = -x
                elif op == SQRT:
                    v = np.sqrt(x)
                elif op == SQ:
                    v = x * x
                elif op == FABS:
                    v = abs(x)
                elif op == FMIN:
                    v = y if x != x else x if y != y else (x if x <= y else y)
                elif op == FMAX:
                    v = y if x != x else x if y != y else (x if x >= y else y)
                elif op == STEP:
                    v = np.float64(1.0) if x > 0 else np.float64(0.0)
                elif op == IF_ELSE:
                    v = np.float64(w[b]) if x != 0 else np.float64(w[c])
                else:
                    raise ValueError(op)
            w[o] = float(v)
    return outs, worst


def explained_by_libm(tape, inputs, rows, gpu_outputs, max_ulps=3, plan_options=None):
    """True iff every listed row's GPU outputs are reproduced by the replay with GPU
    transcendental results, each within ``max_ulps`` of glibc (see the module docstring)."""
    rows = sorted(set(int(r) for r in rows))
    sub = [np.asarray(v)[rows] for v in inputs]
    trace, arith = gpu_trace(tape, sub, plan_options)
    for k, r in enumerate(rows):
        outs, worst = replay_row(tape, [v[k] for v in sub], trace[k], arith)
        if worst > max_ulps:
            return False
        for j, o in enumerate(outs):
            g = np.asarray(gpu_outputs[j])[r]
            same = (o == g) | (np.isnan(o) & np.isnan(g))
            if not same.all():
                return False
    return True
