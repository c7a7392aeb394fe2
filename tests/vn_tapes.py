"""Hand-written tapes for the exact value-numbering pass (csrc/codegen.cpp build_program):
duplicate rows, commuted ADD/MUL operands, FMIN/FMAX operand orders (must NOT be merged:
signed-zero ties keep the first operand, _kernels.py:116-143) and the identities
x*1 = 1*x = x/1 = x-(+0) = x+(-0) = (-0)+x = x, x*(-1) = x/(-1) = -x, -(-x) = x.
Test infrastructure (shared by tests/test_native_cpu.py and tests/test_gpu_parity.py)."""

import numpy as np

from paper_2408_09662_b200 import InstructionTape

CONST, INPUT, OUTPUT, ADD, SUB, MUL, DIV, NEG, FMIN, FMAX = 0, 1, 2, 4, 5, 6, 7, 8, 19, 20

# every IEEE class the identities must hold for: signed zeros, subnormals, infinities, NaN
SPECIALS = np.array([0.0, -0.0, 1.0, -1.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1.5, -2.75,
                     1e308, -1e308, np.inf, -np.inf, np.nan, 3.0, -7.0])


def vn_tape():
    """x, y -> 16 outputs, one per arithmetic row; EXPECTED_CSE of those rows are answered by
    an existing value."""
    rows, vals = [], []

    def row(op, o, a=-1, b=-1, c=-1, v=0.0):
        rows.append([op, o, a, b, c])
        vals.append(v)

    row(INPUT, 0, 0, 0)          # w0 = x
    row(INPUT, 1, 0, 1)          # w1 = y
    row(CONST, 2, v=1.0)
    row(CONST, 3, v=-1.0)
    row(CONST, 4, v=0.0)
    row(CONST, 5, v=-0.0)
    outs = []

    def out(slot):
        outs.append(slot)

    row(MUL, 6, 0, 2); out(6)        # x*1        -> x
    row(MUL, 7, 2, 0); out(7)        # 1*x        -> x
    row(DIV, 8, 0, 2); out(8)        # x/1        -> x
    row(SUB, 9, 0, 4); out(9)        # x-(+0)     -> x
    row(ADD, 10, 0, 5); out(10)      # x+(-0)     -> x
    row(ADD, 11, 5, 0); out(11)      # (-0)+x     -> x
    row(MUL, 12, 0, 3); out(12)      # x*(-1)     -> NEG x (new node)
    row(DIV, 13, 0, 3); out(13)      # x/(-1)     -> the same NEG x
    row(NEG, 14, 12); out(14)        # -(-x)      -> x
    row(ADD, 15, 0, 1); out(15)      # x+y
    row(ADD, 16, 1, 0); out(16)      # y+x        -> x+y
    row(MUL, 17, 0, 1); out(17)      # x*y
    row(MUL, 18, 1, 0); out(18)      # y*x        -> x*y
    row(FMIN, 19, 0, 1); out(19)     # fmin(x,y)
    row(FMIN, 20, 1, 0); out(20)     # fmin(y,x)  kept: ties / NaN order differ
    row(ADD, 21, 0, 4); out(21)      # x+(+0)     kept: -0 + +0 = +0
    for k, s in enumerate(outs):
        row(OUTPUT, 0, s, k)
    return InstructionTape("vn", np.array(rows, dtype=np.int32), np.array(vals), 22, [2], [len(outs)])


# rows answered by an existing value: x*1, 1*x, x/1, x-0, x+(-0), (-0)+x, x/(-1) (same NEG as
# x*(-1)), -(-x), y+x, y*x
EXPECTED_CSE = 10


def vn_inputs():
    a, b = np.meshgrid(SPECIALS, SPECIALS, indexing="ij")
    return [np.stack([a.ravel(), b.ravel()], axis=1)]
