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
