"""Instruction-tape ingest: the IR the batched evaluator consumes.

This is the host-side mirror of the reference's tape layer
(``vecsym.tape``, /root/reference/pkg/src/vecsym/tape.py) restricted to what
the hot path needs: the packed tape object, its validation, and the
``"vecsym-tape"`` v1 text format.  Graph building and ``flatten`` stay in the
reference (they are offline tape *producers*).

Wire format of one row (tape.py:10-20): ``[op, out, in0, in1, in2]`` int32
plus one float64 ``value``; unused fields hold -1.

    CONST   out=work slot            value = constant
    INPUT   out=work slot            in0 = input index,  in1 = nonzero ordinal
    OUTPUT  out=output index         in0 = source slot,  in1 = nonzero ordinal
    others  out=work slot            in0..in2 = operand slots (arity-many)
"""

from __future__ import annotations

import enum
import gzip
import json
from typing import Sequence

import numpy as np

__all__ = [
    "OpCode",
    "ARITY",
    "arity",
    "Sparsity",
    "InstructionTape",
    "as_tape",
    "serialize",
    "deserialize",
    "save",
    "load",
    "FORMAT_VERSION",
    "PLUMBING_OPS",
]

FORMAT_VERSION = 1


class OpCode(enum.IntEnum):
    """Opcode wire values (symcore.py:72-97)."""

    CONST = 0
    INPUT = 1
    OUTPUT = 2
    ASSIGN = 3
    ADD = 4
    SUB = 5
    MUL = 6
    DIV = 7
    NEG = 8
    EXP = 9
    LOG = 10
    POW = 11
    SQRT = 12
    SQ = 13
    SIN = 14
    COS = 15
    TAN = 16
    ATAN2 = 17
    FABS = 18
    FMIN = 19
    FMAX = 20
    STEP = 21
    IF_ELSE = 22


# operand counts (symcore.py:100-124); indexed by wire value
ARITY = np.array([0, 0, 1, 1, 2, 2, 2, 2, 1, 1, 1, 2, 1, 1, 1, 1, 1, 2, 1, 2, 2, 1, 3], dtype=np.int64)

# rows that move data rather than compute (bench.py:50-52)
PLUMBING_OPS = (OpCode.CONST, OpCode.INPUT, OpCode.OUTPUT, OpCode.ASSIGN)


def arity(op) -> int:
    return int(ARITY[int(OpCode(op))])


class Sparsity:
    """Compressed-column pattern; nonzero ordinal k is column-major
    (symcore.py:296-301).  Only the shape data the evaluator needs."""

    __slots__ = ("rows", "cols", "colptr", "rowidx")

    def __init__(self, rows: int, cols: int, colptr: Sequence[int], rowidx: Sequence[int]):
        rows, cols = int(rows), int(cols)
        colptr = tuple(int(p) for p in colptr)
        rowidx = tuple(int(r) for r in rowidx)
        if rows < 0 or cols < 0:
            raise ValueError("negative dimension")
        if len(colptr) != cols + 1 or colptr[0] != 0 or colptr[-1] != len(rowidx):
            raise ValueError("malformed column pointer")
        cp = np.asarray(colptr, dtype=np.int64)
        if np.any(np.diff(cp) < 0):
            raise ValueError("column pointer not non-decreasing")
        ri = np.asarray(rowidx, dtype=np.int64)
        if ri.size and (ri.min() < 0 or ri.max() >= rows):
            bad = int(ri[(ri < 0) | (ri >= rows)][0])
            raise ValueError(f"row index {bad} out of range for {rows} rows")
        for c in range(cols):
            seg = ri[cp[c] : cp[c + 1]]
            if seg.size > 1 and np.any(np.diff(seg) <= 0):
                raise ValueError("row indices must strictly increase within a column")
        self.rows, self.cols, self.colptr, self.rowidx = rows, cols, colptr, rowidx

    @staticmethod
    def dense(rows: int, cols: int = 1) -> "Sparsity":
        return Sparsity(rows, cols, [c * rows for c in range(cols + 1)], [r for _ in range(cols) for r in range(rows)])

    @property
    def nnz(self) -> int:
        return len(self.rowidx)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    def to_obj(self) -> dict:
        return {"rows": self.rows, "cols": self.cols, "colptr": list(self.colptr), "rowidx": list(self.rowidx)}

    def __eq__(self, other) -> bool:
        return (
            isinstance(other, Sparsity)
            and (self.rows, self.cols, self.colptr, self.rowidx)
            == (other.rows, other.cols, other.colptr, other.rowidx)
        )

    def __hash__(self) -> int:
        return hash((self.rows, self.cols, self.colptr, self.rowidx))

    def __repr__(self) -> str:
        return f"Sparsity({self.rows}x{self.cols}, {self.nnz} nnz)"


def _coerce_sparsity(sp) -> Sparsity:
    if isinstance(sp, Sparsity):
        return sp
    if isinstance(sp, (int, np.integer)):
        return Sparsity.dense(int(sp), 1)
    # duck-typed reference vecsym.symcore.Sparsity
    return Sparsity(sp.rows, sp.cols, sp.colptr, sp.rowidx)


class TapeError(ValueError):
    """Validation failure; the message names the offending row."""


def _row_error(i: int, msg: str) -> TapeError:
    return TapeError(f"instruction {i}: {msg}")


class InstructionTape:
    """Validated packed tape (the reference's ``InstructionTape``, tape.py:80-123).

    ``input_sparsity`` / ``output_sparsity`` accept Sparsity objects (ours or
    the reference's) or plain ints (dense column vectors of that length).
    """

    __slots__ = ("name", "format_version", "n_w", "input_sparsity", "output_sparsity",
                 "_code", "_values", "_digest")

    def __init__(self, name, code, values, n_w, input_sparsity, output_sparsity):
        if not str(name).isidentifier():
            raise ValueError(f"tape name {name!r} is not a valid identifier")
        code = np.ascontiguousarray(np.asarray(code, dtype=np.int32).reshape(-1, 5))
        values = np.ascontiguousarray(np.asarray(values, dtype=np.float64).ravel())
        if values.shape[0] != code.shape[0]:
            raise ValueError("code and value arrays disagree on instruction count")
        code.setflags(write=False)
        values.setflags(write=False)
        self.name = str(name)
        self.format_version = FORMAT_VERSION
        self.n_w = int(n_w)
        self.input_sparsity = [_coerce_sparsity(s) for s in input_sparsity]
        self.output_sparsity = [_coerce_sparsity(s) for s in output_sparsity]
        self._code = code
        self._values = values
        self._digest = None
        validate(self)

    @property
    def n_instructions(self) -> int:
        return int(self._code.shape[0])

    @property
    def nnz_in(self) -> list[int]:
        return [s.nnz for s in self.input_sparsity]

    @property
    def nnz_out(self) -> list[int]:
        return [s.nnz for s in self.output_sparsity]

    @property
    def n_in(self) -> int:
        return len(self.input_sparsity)

    @property
    def n_out(self) -> int:
        return len(self.output_sparsity)

    def packed(self) -> tuple[np.ndarray, np.ndarray]:
        """(int32 [n,5] code, float64 [n] values), read-only (tape.py:159-161)."""
        return self._code, self._values

    @property
    def n_arith(self) -> int:
        """Arithmetic rows: everything but CONST/INPUT/OUTPUT/ASSIGN (bench.py:50-52,117)."""
        ops = self._code[:, 0]
        return int(np.count_nonzero(~np.isin(ops, [int(o) for o in PLUMBING_OPS])))

    def digest(self) -> str:
        """Content hash (code, values, shapes) used as the compile-cache key."""
        if self._digest is None:
            import hashlib

            h = hashlib.sha256()
            h.update(self._code.tobytes())
            h.update(self._values.tobytes())
            h.update(np.asarray([self.n_w] + self.nnz_in + [-1] + self.nnz_out, dtype=np.int64).tobytes())
            self._digest = h.hexdigest()
        return self._digest

    def __repr__(self) -> str:
        return (f"InstructionTape({self.name!r}, {self.n_instructions} instructions, "
                f"n_w={self.n_w}, nnz_in={self.nnz_in}, nnz_out={self.nnz_out})")


def validate(t: InstructionTape) -> None:
    """Structural checks of tape.py:171-258: known opcodes, index ranges,
    -1 sentinels in unused fields, and every work slot written before it is
    read.  Row order is otherwise free (INPUT/OUTPUT rows may interleave)."""
    code = t._code
    n = code.shape[0]
    if t.n_w < 0:
        raise ValueError("n_w must be nonnegative")
    if n == 0:
        return
    op = code[:, 0].astype(np.int64)
    unknown = (op < 0) | (op > int(OpCode.IF_ELSE))
    if unknown.any():
        i = int(np.flatnonzero(unknown)[0])
        raise _row_error(i, f"unknown opcode {int(op[i])}")
    out, a, b, c = (code[:, k].astype(np.int64) for k in (1, 2, 3, 4))
    k_const = op == OpCode.CONST
    k_input = op == OpCode.INPUT
    k_output = op == OpCode.OUTPUT
    k_work = ~(k_const | k_input | k_output)
    ar = np.where(k_work, ARITY[op], 0)
    nnz_in = np.asarray(t.nnz_in or [0], dtype=np.int64)
    nnz_out = np.asarray(t.nnz_out or [0], dtype=np.int64)
    n_w, n_in, n_out = t.n_w, t.n_in, t.n_out

    checks = []  # (mask, message) evaluated in order; first failing row wins per check
    checks.append(((k_const | k_input | k_work) & ((out < 0) | (out >= n_w)), f"work index out of range (n_w={n_w})"))
    checks.append((k_output & ((n_out == 0) | (out < 0) | (out >= max(n_out, 1))), f"output index out of range ({n_out} outputs)"))
    checks.append((k_input & ((n_in == 0) | (a < 0) | (a >= max(n_in, 1))), f"input index out of range ({n_in} inputs)"))
    checks.append((k_input & ((b < 0) | (b >= nnz_in[np.clip(a, 0, max(n_in - 1, 0))])), "nonzero offset out of range for input"))
    checks.append((k_output & ((b < 0) | (b >= nnz_out[np.clip(out, 0, max(n_out - 1, 0))])), "nonzero offset out of range for output"))
    checks.append((k_output & ((a < 0) | (a >= n_w)), f"work index out of range (n_w={n_w})"))
    for mask, msg in checks:
        if mask.any():
            raise _row_error(int(np.flatnonzero(mask)[0]), msg)
    fields = (a, b, c)
    for k in range(3):
        used = k_work & (ar > k)
        bad = used & ((fields[k] < 0) | (fields[k] >= n_w))
        if bad.any():
            raise _row_error(int(np.flatnonzero(bad)[0]), f"work index out of range (n_w={n_w})")
        bad = k_work & (ar <= k) & (fields[k] != -1)
        if bad.any():
            raise _row_error(int(np.flatnonzero(bad)[0]), "expected -1 sentinel in unused field")
    bad = k_const & ((a != -1) | (b != -1) | (c != -1))
    if bad.any():
        raise _row_error(int(np.flatnonzero(bad)[0]), "expected -1 sentinels for CONST")
    bad = (k_input | k_output) & (c != -1)
    if bad.any():
        raise _row_error(int(np.flatnonzero(bad)[0]), "expected -1 sentinel in unused field")

    # write-before-read: a read at row r of slot s needs some writer of s at row < r
    rows = np.arange(n, dtype=np.int64)
    first_write = np.full(max(n_w, 1), n, dtype=np.int64)
    w = ~k_output
    np.minimum.at(first_write, out[w], rows[w])
    rd_rows = [rows[k_output]]
    rd_slots = [a[k_output]]
    for k in range(3):
        m = k_work & (ar > k)
        rd_rows.append(rows[m])
        rd_slots.append(fields[k][m])
    rr = np.concatenate(rd_rows)
    rs = np.concatenate(rd_slots)
    if rr.size:
        early = first_write[rs] >= rr
        if early.any():
            raise _row_error(int(rr[early].min()), "work slot read before any write")


def as_tape(obj) -> InstructionTape:
    """Accept our tape, a reference ``vecsym`` InstructionTape (duck-typed on
    ``packed()``), or a path to a ``.tape.json[.gz]`` file."""
    if isinstance(obj, InstructionTape):
        return obj
    if isinstance(obj, (str, bytes)) or hasattr(obj, "__fspath__"):
        return load(obj)
    if hasattr(obj, "packed") and hasattr(obj, "input_sparsity"):
        code, values = obj.packed()
        return InstructionTape(obj.name, code, values, obj.n_w, obj.input_sparsity, obj.output_sparsity)
    raise TypeError(f"cannot interpret {type(obj).__name__} as an instruction tape")


# ---------------------------------------------------------------------------
# "vecsym-tape" v1 text format (tape.py:387-457)
# ---------------------------------------------------------------------------

_OPNAMES = [o.name for o in OpCode]
_BY_NAME = {o.name: int(o) for o in OpCode}


def serialize(t: InstructionTape) -> str:
    """Line-oriented JSON text, one row per line; byte-compatible with the
    reference's serializer so files round-trip between the two."""
    code, values = t.packed()
    parts = [
        "{",
        '"format": "vecsym-tape",',
        f'"format_version": {t.format_version},',
        f'"name": {json.dumps(t.name)},',
        f'"n_w": {t.n_w},',
        f'"n_instructions": {t.n_instructions},',
        f'"input_sparsity": {json.dumps([s.to_obj() for s in t.input_sparsity])},',
        f'"output_sparsity": {json.dumps([s.to_obj() for s in t.output_sparsity])},',
        '"columns": ["op", "out", "in0", "in1", "in2", "value"],',
        '"instructions": [',
    ]
    n = code.shape[0]
    body = []
    for i, (row, v) in enumerate(zip(code.tolist(), values.tolist())):
        sep = "," if i + 1 < n else ""
        body.append(f'["{_OPNAMES[row[0]]}", {row[1]}, {row[2]}, {row[3]}, {row[4]}, {json.dumps(v)}]{sep}')
    return "\n".join(parts + body + ["]", "}"]) + "\n"


def deserialize(text: str) -> InstructionTape:
    """Parse + validate; diagnostics name the offending row (tape.py:412-457)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ValueError(f"not a tape file: invalid JSON ({e})") from None
    if not isinstance(doc, dict) or doc.get("format") != "vecsym-tape":
        raise ValueError("not a tape file: missing 'vecsym-tape' format marker")
    if doc.get("format_version") != FORMAT_VERSION:
        raise ValueError(
            f"unsupported tape format_version {doc.get('format_version')!r} (this build reads {FORMAT_VERSION})"
        )
    for key in ("name", "n_w", "n_instructions", "input_sparsity", "output_sparsity", "instructions"):
        if key not in doc:
            raise ValueError(f"not a tape file: missing field {key!r}")

    def sp(obj, what):
        try:
            return Sparsity(obj["rows"], obj["cols"], obj["colptr"], obj["rowidx"])
        except (KeyError, TypeError, ValueError) as e:
            raise ValueError(f"malformed {what} sparsity: {e}") from None

    ins = [sp(o, f"input {i}") for i, o in enumerate(doc["input_sparsity"])]
    outs = [sp(o, f"output {i}") for i, o in enumerate(doc["output_sparsity"])]
    rows = doc["instructions"]
    if not isinstance(rows, list):
        raise ValueError("instructions must be a list")
    if len(rows) != doc["n_instructions"]:
        raise ValueError(f"n_instructions is {doc['n_instructions']} but {len(rows)} rows are present")
    n = len(rows)
    code = np.empty((n, 5), dtype=np.int32)
    values = np.zeros(n, dtype=np.float64)
    for i, row in enumerate(rows):
        if not isinstance(row, list) or len(row) != 6:
            raise _row_error(i, "expected a 6-field row [op, out, in0, in1, in2, value]")
        opnum = _BY_NAME.get(row[0]) if isinstance(row[0], str) else None
        if opnum is None:
            raise _row_error(i, f"unknown opcode {row[0]!r}")
        for k in range(1, 5):
            if not isinstance(row[k], int):
                raise _row_error(i, f"index field {k} must be an integer, got {row[k]!r}")
        if not isinstance(row[5], (int, float)):
            raise _row_error(i, f"value field must be a number, got {row[5]!r}")
        code[i] = (opnum, row[1], row[2], row[3], row[4])
        values[i] = float(row[5])
    if not isinstance(doc["name"], str):
        raise ValueError("tape name must be a string")
    return InstructionTape(doc["name"], code, values, int(doc["n_w"]), ins, outs)


def save(t: InstructionTape, path) -> None:
    path = str(path)
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "wt", encoding="utf-8") as fh:
        fh.write(serialize(t))


def load(path) -> InstructionTape:
    path = str(path if not isinstance(path, bytes) else path.decode())
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        return deserialize(fh.read())
