import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# transcendental-free ops must be bit-identical to the reference CPU path
EXACT_OPS = ("ASSIGN", "ADD", "SUB", "MUL", "DIV", "NEG", "SQRT", "SQ", "FABS", "FMIN", "FMAX", "STEP", "IF_ELSE")
# fp64 parity contract (BASELINE.json north_star): 1e-12 relative, NaN == NaN
RTOL64 = 1e-12
# fp32 mode contract: 1e-4 relative to max(|ref|, 1)
RTOL32 = 1e-4


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise_or_nan(got, ref, what=""):
    """Bit-identical on every non-NaN value; NaN matches any NaN (the
    reference's own serial and batched paths disagree on NaN sign bits)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    both_nan = np.isnan(got) & np.isnan(ref)
    bad = (bits(got) != bits(ref)) & ~both_nan
    assert not bad.any(), f"{what}: {int(bad.sum())} mismatches, first at {np.argwhere(bad)[0]}: got {got[bad][0]!r} ref {ref[bad][0]!r}"


def close_mask(got, ref, rtol):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    both_nan = np.isnan(got) & np.isnan(ref)
    same = (got == ref) | both_nan
    with np.errstate(invalid="ignore", over="ignore"):
        err = np.abs(got - ref)
        tol = rtol * np.maximum(np.abs(ref), 1.0)
        ok = same | (np.isfinite(ref) & np.isfinite(got) & (err <= tol))
    return ok


def assert_close(got, ref, rtol=RTOL64, what=""):
    """|g - r| <= rtol * max(|r|, 1); NaN == NaN; infinities must match exactly."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    ok = close_mask(got, ref, rtol)
    if not ok.all():
        idx = np.argwhere(~ok)[0]
        raise AssertionError(
            f"{what}: {int((~ok).sum())}/{ok.size} outside rtol={rtol}; first at {tuple(idx)}: "
            f"got {got[tuple(idx)]!r} ref {ref[tuple(idx)]!r}"
        )


def assert_parity(got, ref, spread=None, rtol=RTOL64, what="", factor=4.0):
    """The fp64 parity contract: |g - r| <= max(rtol * max(|r|, 1), factor * spread)
    where ``spread`` is the reference algorithm's own deviation when its
    transcendental results move by the ulps two conforming libms may differ by
    (oracle.sensitivity: 1 for sin/cos, 2 for exp/log, 3 for pow/tan/atan2; zero for
    transcendental-free tapes, which therefore must match to 1e-12 -- and are
    in fact bit-identical).  NaN == NaN, infinities exact."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    ok = close_mask(got, ref, rtol)
    if spread is not None:
        with np.errstate(invalid="ignore"):
            ok |= np.isfinite(got) & np.isfinite(ref) & (np.abs(got - ref) <= factor * np.asarray(spread))
    if not ok.all():
        idx = tuple(np.argwhere(~ok)[0])
        sp = float(np.asarray(spread)[idx]) if spread is not None else 0.0
        raise AssertionError(
            f"{what}: {int((~ok).sum())}/{ok.size} outside contract; first at {idx}: got {got[idx]!r} "
            f"ref {ref[idx]!r} (1-ulp-libm spread {sp:.3g})"
        )


@pytest.fixture(scope="session")
def golden_ops():
    return np.load(os.path.join(GOLDEN, "ops_specials.npz"))


@pytest.fixture(scope="session")
def golden_random():
    return np.load(os.path.join(GOLDEN, "random_tapes.npz"))


@pytest.fixture(scope="session")
def golden_workloads():
    return np.load(os.path.join(GOLDEN, "workloads.npz"))
