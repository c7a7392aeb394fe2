"""Tape ingest: the vecsym-tape v1 format and validation (tape.py:171-258,387-457)."""

import gzip

import numpy as np
import pytest

import workloads
from paper_2408_09662_b200.tape import InstructionTape, OpCode, Sparsity, as_tape, deserialize, load, save, serialize


def test_serialize_is_byte_identical_to_reference_files():
    # every workloads/*.tape.json.gz was written by the reference serializer
    for name in workloads.NAMES:
        with gzip.open(workloads.tape_path(name), "rt", encoding="utf-8") as fh:
            text = fh.read()
        assert serialize(deserialize(text)) == text, name


def test_fig2_tape_rows():
    t = workloads.load_tape("example")
    assert t.n_instructions == 5 and t.n_w == 2
    code, _ = t.packed()
    assert [OpCode(r[0]).name for r in code] == ["INPUT", "SIN", "ADD", "MUL", "OUTPUT"]


def test_round_trip_file(tmp_path):
    t = workloads.load_tape("cartpole_rk4")
    for fname in ("c.tape.json", "c.tape.json.gz"):
        save(t, tmp_path / fname)
        u = load(tmp_path / fname)
        assert np.array_equal(u.packed()[0], t.packed()[0])
        assert np.array_equal(u.packed()[1].view(np.uint64), t.packed()[1].view(np.uint64))
        assert u.nnz_in == t.nnz_in and u.nnz_out == t.nnz_out and u.n_w == t.n_w


def test_packed_is_read_only():
    code, values = workloads.load_tape("pendulum").packed()
    with pytest.raises(ValueError):
        code[0, 0] = 3
    with pytest.raises(ValueError):
        values[0] = 1.0


def _tape(rows, n_w=2, nin=(1,), nout=(1,), values=None):
    rows = np.array(rows, dtype=np.int32)
    return InstructionTape("t", rows, np.zeros(len(rows)) if values is None else values, n_w, list(nin), list(nout))


@pytest.mark.parametrize(
    "rows, msg",
    [
        ([[1, 0, 0, 0, -1], [99, 0, 0, -1, -1]], "instruction 1: unknown opcode 99"),
        ([[1, 5, 0, 0, -1]], r"instruction 0: work index out of range \(n_w=2\)"),
        ([[1, 0, 3, 0, -1]], r"instruction 0: input index out of range \(1 inputs\)"),
        ([[1, 0, 0, 4, -1]], "instruction 0: nonzero offset out of range for input"),
        ([[1, 0, 0, 0, -1], [2, 2, 0, 0, -1]], r"instruction 1: output index out of range \(1 outputs\)"),
        ([[1, 0, 0, 0, -1], [2, 0, 0, 7, -1]], "instruction 1: nonzero offset out of range for output"),
        ([[1, 0, 0, 0, -1], [4, 1, 0, 1, -1]], "instruction 1: work slot read before any write"),
        ([[1, 0, 0, 0, -1], [8, 1, 0, 0, -1]], "instruction 1: expected -1 sentinel in unused field"),
        ([[0, 0, 1, -1, -1]], "instruction 0: expected -1 sentinels for CONST"),
        ([[1, 0, 0, 0, 0]], "instruction 0: expected -1 sentinel in unused field"),
    ],
)
def test_validation_messages(rows, msg):
    with pytest.raises(ValueError, match=msg):
        _tape(rows)


def test_deserialize_errors():
    with pytest.raises(ValueError, match="invalid JSON"):
        deserialize("{")
    with pytest.raises(ValueError, match="missing 'vecsym-tape' format marker"):
        deserialize('{"format": "x"}')
    with pytest.raises(ValueError, match="unsupported tape format_version 2"):
        deserialize('{"format": "vecsym-tape", "format_version": 2}')
    text = serialize(workloads.load_tape("example"))
    with pytest.raises(ValueError, match="instruction 1: unknown opcode 'FOO'"):
        deserialize(text.replace('["SIN"', '["FOO"'))
    with pytest.raises(ValueError, match="n_instructions is 5 but 4 rows"):
        deserialize(text.replace('["SIN", 1, 0, -1, -1, 0.0],\n', ""))


def test_sparsity_checks():
    assert Sparsity.dense(3, 2).nnz == 6
    with pytest.raises(ValueError, match="malformed column pointer"):
        Sparsity(2, 1, [0], [])
    with pytest.raises(ValueError, match="strictly increase"):
        Sparsity(3, 1, [0, 2], [1, 1])


def test_as_tape_accepts_duck_typed_reference_objects():
    t = workloads.load_tape("pendulum")

    class RefLike:
        name = t.name
        n_w = t.n_w
        input_sparsity = t.input_sparsity
        output_sparsity = t.output_sparsity

        def packed(self):
            return t.packed()

    u = as_tape(RefLike())
    assert u.digest() == t.digest()
    assert as_tape(workloads.tape_path("pendulum")).digest() == t.digest()


def test_arith_count_matches_bench_definition():
    # bench.py:50-52,117 counts everything but CONST/INPUT/OUTPUT/ASSIGN
    t = workloads.load_tape("srbm_mpc")
    code, _ = t.packed()
    plumbing = np.isin(code[:, 0], [0, 1, 2, 3])
    assert t.n_arith == int((~plumbing).sum()) == 111153
