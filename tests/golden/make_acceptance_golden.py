"""Acceptance-criterion-1 fuzz goldens, made by running the REFERENCE itself.

Dev-container only (``source tools/refenv.sh`` first).  Mirrors the tape plan
of the reference's acceptance criterion 1
(/root/reference/pkg/tests/test_acceptance.py:69-111): 100 tapes from the
reference fuzzer ``random_tape_function`` (tests/oracles.py:208-269), rng
``random.Random(20260814)``, sizes ``geomspace(12, 48000, 100)`` shrunk by 0.7
until the flattened tape has <= 10,000 instructions.  These tapes reach the
sizes where this build's team scheduler (>= 4000 live ops), cross-warp
shared-memory slots, overflow scratch and the chunk splitter engage.

A second family, ``exact``, uses the same generator shape over the
transcendental-free opcodes only (ADD SUB MUL DIV NEG SQRT SQ FABS FMIN FMAX
STEP IF_ELSE ASSIGN): for those tapes every GPU result must be bit-identical
to the reference, at every size and in every kernel regime.

Inputs: U[-2, 2] per element from ``np.random.default_rng(SEED + idx)`` (the
tests regenerate them; only the first ``ROWS`` rows' reference outputs are
stored).  Output: tests/golden/acceptance.npz
  {fam}{idx}__tape   uint8: the reference serializer's "vecsym-tape" v1 text
  {fam}{idx}__out{j} float64 [ROWS, nnz_out[j]]: reference batch_eval outputs
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from vecsym import symcore as sc  # noqa: E402
from vecsym.batchrt import BatchWorkspace, batch_eval, serial_eval  # noqa: E402
from vecsym.tape import flatten, serialize  # noqa: E402
from oracles import random_tape_function  # noqa: E402  (reference tests/oracles.py)

SEED = {"acc": 5000, "exact": 6000}
ROWS = 64
MAX_INSTR = 10_000


def inputs_for(fam: str, idx: int, nnz_in, batch: int):
    """The per-element inputs the tests regenerate (U[-2, 2], seeded per tape)."""
    rng = np.random.default_rng(SEED[fam] + idx)
    return [rng.uniform(-2.0, 2.0, size=(batch, n)) for n in nnz_in]


def exact_tape_function(rng: random.Random, name: str, n_ops: int):
    """Random DAG over the transcendental-free opcodes (same growth rule as the
    reference fuzzer: half the operands drawn from the 8 newest nodes)."""
    Op = sc.OpCode
    n_inputs = rng.randint(1, 3)
    syms = [sc.sym(f"x{i}", rng.randint(1, 5)) for i in range(n_inputs)]
    pool = [s[k] for s in syms for k in range(s.rows)]
    for _ in range(2):
        pool.append(sc.constant(round(rng.uniform(-2.0, 2.0), 3)))
    unary = [Op.NEG, Op.SQRT, Op.SQ, Op.FABS, Op.STEP, Op.ASSIGN]
    binary = [Op.ADD, Op.SUB, Op.MUL, Op.DIV, Op.FMIN, Op.FMAX]

    def pick():
        if rng.random() < 0.5 and len(pool) > 8:
            return pool[rng.randrange(len(pool) - 8, len(pool))]
        return pool[rng.randrange(len(pool))]

    for _ in range(n_ops):
        kind = rng.random()
        if kind < 0.3:
            pool.append(sc.apply(rng.choice(unary), pick()))
        elif kind < 0.9:
            pool.append(sc.apply(rng.choice(binary), pick(), pick()))
        else:
            pool.append(sc.if_else(pick(), pick(), pick()))
    n_out = rng.randint(1, 3)
    outs = []
    tail = pool[-(4 * n_out):]
    step = max(1, len(tail) // n_out)
    for oi in range(n_out):
        outs.append(sc.vertcat(tail[oi * step:(oi + 1) * step] or [pool[-1]]))
    return sc.SymbolicFunction(name, syms, outs)


def make(fam: str, gen, seed: int):
    rng = random.Random(seed)
    out = {}
    sizes = []
    for idx, n_ops in enumerate(int(n) for n in np.geomspace(12, 48_000, 100)):
        tape = flatten(gen(rng, name=f"{fam}{idx}", n_ops=n_ops))
        while tape.n_instructions > MAX_INSTR:
            n_ops = int(n_ops * 0.7)
            tape = flatten(gen(rng, name=f"{fam}{idx}", n_ops=n_ops))
        sizes.append(tape.n_instructions)
        ins = inputs_for(fam, idx, tape.nnz_in, ROWS)
        ws = BatchWorkspace(tape, ROWS)
        for i, v in enumerate(ins):
            ws.set_input(i, v)
        batch_eval(tape, ws, n_threads=1)
        # the reference's own criterion: batch == serial bit for bit (checked on 4 rows here)
        for e in (0, 1, ROWS // 2, ROWS - 1):
            ser = serial_eval(tape, [v[e] for v in ins])
            for j in range(tape.n_out):
                a = np.ascontiguousarray(ser[j]).view(np.uint64)
                b = np.ascontiguousarray(ws.output_matrix(j)[e]).view(np.uint64)
                nan = np.isnan(ser[j]) & np.isnan(ws.output_matrix(j)[e])
                assert ((a == b) | nan).all(), (fam, idx, e, j)
        out[f"{fam}{idx}__tape"] = np.frombuffer(serialize(tape).encode(), dtype=np.uint8)
        for j in range(tape.n_out):
            out[f"{fam}{idx}__out{j}"] = ws.output_matrix(j).copy()
    print(fam, "sizes", min(sizes), max(sizes), "sum", sum(sizes), flush=True)
    return out


if __name__ == "__main__":
    d = {}
    d.update(make("acc", random_tape_function, 20260814))
    d.update(make("exact", exact_tape_function, 20261017))
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **d)
