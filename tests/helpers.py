"""Test helpers (bit-exact comparisons)."""
import numpy as np
import pytest


def bits(a) -> np.ndarray:
    """float64 array -> uint64 bit patterns."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def hex_to_bits(lst) -> np.ndarray:
    return np.array([int(h, 16) for h in lst], dtype=np.uint64)


def assert_bits_equal(got, want, what=""):
    g, w = bits(got), np.asarray(want, dtype=np.uint64)
    assert g.shape == w.shape, f"{what}: shape {g.shape} vs {w.shape}"
    bad = np.flatnonzero(g != w)
    if bad.size:
        i = int(bad[0])
        pytest.fail(f"{what}: {bad.size} mismatches, first at {i}: "
                    f"{g.view(np.float64)[i]!r} vs {w.view(np.float64)[i]!r}")


def ulp_diff(a, b) -> np.ndarray:
    """|a - b| in units of the last place (ordered bit patterns of float64)."""
    def ordered(x):
        u = bits(x).astype(np.int64)
        return np.where(u < 0, np.int64(-2**63) - u, u)
    return np.abs(ordered(a) - ordered(b))


def assert_trad_close(got, want, tail_mask, what=""):
    """Traditional samplers: bit equality everywhere except tail samples
    (their value is a libm log), which may differ by at most 2 ulp."""
    g, w = bits(got), np.asarray(want, dtype=np.uint64)
    assert g.shape == w.shape, f"{what}: shape {g.shape} vs {w.shape}"
    bad = np.flatnonzero(g != w)
    if bad.size:
        tail = np.asarray(tail_mask, dtype=bool)
        assert tail[bad].all(), f"{what}: non-tail mismatch at {bad[~tail[bad]][:5]}"
        d = ulp_diff(g[bad].view(np.float64), w[bad].view(np.float64))
        assert d.max() <= 2, f"{what}: tail sample off by {d.max()} ulp"
