"""Generate golden vectors by running the REFERENCE evaluator itself.

Dev-container only (imports the read-only reference; ``source
tools/refenv.sh`` first).  Produces small committed fixtures that pin the
oracle (``oracle/``) and the GPU parity tests to the reference's own
outputs:

  ops_specials.npz   every evaluable opcode on the reference's SPECIALS grid
                     (tests/test_batchrt.py:21-30,52-81) + seeded randoms,
                     outputs from vecsym.batchrt.batch_eval (numba run_range)
  random_tapes.npz   40 random tapes from tests/oracles.py:208-269, B=64 each
  workloads.npz      every workloads/*.tape.json.gz at a small batch with
                     workloads.make_inputs inputs

Every output is the reference's ``batch_eval`` result; the same cases were
checked against ``serial_eval`` by the reference's own tests.
"""

from __future__ import annotations

import math
import os
import random
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from vecsym.batchrt import BatchWorkspace, batch_eval  # noqa: E402
from vecsym.symcore import OpCode, SymbolicFunction, apply, arity, sym  # noqa: E402
from vecsym.tape import flatten, serialize  # noqa: E402
from oracles import random_tape_function  # noqa: E402  (reference tests/oracles.py)

import workloads  # noqa: E402

NEG_NAN = struct.unpack("<d", bytes.fromhex("000000000000f8ff"))[0]
SPECIALS = [
    0.0, -0.0, 1.0, -1.0, 0.5, -0.5, 2.0, -2.0, 3.0, -3.0, 0.75, -0.75,
    1.5, -1.5, math.pi, -math.pi, 1e-300, -1e-300, 5e-324, -5e-324,
    1e300, -1e300, 708.5, -745.5, 1e9, -1e9, 1e9 + 1.0, -(1e9 + 1.0),
    float("inf"), float("-inf"), float("nan"), NEG_NAN,
]
EVAL_OPS = [op for op in OpCode if op not in (OpCode.CONST, OpCode.INPUT, OpCode.OUTPUT)]


def ref_eval(tape, inputs):
    B = inputs[0].shape[0] if inputs else 1
    ws = BatchWorkspace(tape, B)
    for i, v in enumerate(inputs):
        ws.set_input(i, v)
    batch_eval(tape, ws, n_threads=1)
    return [ws.output_matrix(j).copy() for j in range(tape.n_out)]


def ops_specials():
    out = {}
    for op in EVAL_OPS:
        n = arity(op)
        rng = np.random.default_rng(1000 + int(op))
        if n == 1:
            cases = [(a,) for a in SPECIALS]
        elif n == 2:
            cases = [(a, b) for a in SPECIALS for b in SPECIALS]
        else:
            sub = SPECIALS[::3]
            cases = [(a, b, c) for a in SPECIALS for b in sub for c in sub]
        randoms = rng.uniform(-50.0, 50.0, size=(500, n))
        randoms[::5] *= 1e30
        randoms[3::5] *= 1e-30
        arr = np.array(cases + [tuple(r) for r in randoms], dtype=np.float64)
        ins = [sym(f"x{k}", 1) for k in range(n)]
        tape = flatten(SymbolicFunction("probe", ins, [apply(op, *ins)]))
        (res,) = ref_eval(tape, [arr[:, k : k + 1] for k in range(n)])
        out[f"{op.name}__tape"] = np.array(serialize(tape))
        out[f"{op.name}__x"] = arr
        out[f"{op.name}__y"] = res[:, 0]
    np.savez_compressed(os.path.join(HERE, "ops_specials.npz"), **out)


def random_tapes(n_tapes=40, B=64):
    out = {}
    rng = random.Random(20240817)
    for t in range(n_tapes):
        f = random_tape_function(rng, name=f"rt{t}", n_ops=rng.randint(5, 400))
        tape = flatten(f)
        # per-element inputs drawn like random_input_values (U[-2,2], oracles.py:272-277)
        ins = [np.array([[rng.uniform(-2.0, 2.0) for _ in range(m.nnz)] for _ in range(B)]) for m in f.inputs]
        outs = ref_eval(tape, ins)
        out[f"t{t}__tape"] = np.array(serialize(tape))
        for i, v in enumerate(ins):
            out[f"t{t}__in{i}"] = v
        for j, v in enumerate(outs):
            out[f"t{t}__out{j}"] = v
    np.savez_compressed(os.path.join(HERE, "random_tapes.npz"), **out)


WORKLOAD_BATCH = {
    "example": 64, "pendulum": 256, "cartpole_rk4": 1000, "ldlt_12": 64, "ldlt_25": 16,
    "ldlt_57": 4, "quad_step": 16, "unicycle_mpc": 8, "srbm_mpc": 8, "rbd_chain12": 4,
    "humanoid_rbd": 16,
}


def workload_goldens():

    out = {}
    for name, B in WORKLOAD_BATCH.items():
        tape = ref_load_gz(workloads.tape_path(name))
        ins = workloads.make_inputs(name, B, seed=123)
        outs = ref_eval(tape, ins)
        for i, v in enumerate(ins):
            out[f"{name}__in{i}"] = v
        for j, v in enumerate(outs):
            out[f"{name}__out{j}"] = v
        print(name, B, [o.shape for o in outs], flush=True)
    np.savez_compressed(os.path.join(HERE, "workloads.npz"), **out)


def ref_load_gz(path):
    import gzip

    from vecsym.tape import deserialize

    with gzip.open(path, "rt", encoding="utf-8") as fh:
        return deserialize(fh.read())


if __name__ == "__main__":
    which = sys.argv[1:] or ["ops", "random", "workloads"]
    if "ops" in which:
        ops_specials()
    if "random" in which:
        random_tapes()
    if "workloads" in which:
        workload_goldens()
