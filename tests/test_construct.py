"""Table construction: the Newton-based solver rebuilds the
reference's shipped i_max = 256 fixtures -- same layer count and heights,
edges to the last bit except where the layer equation changes sign more than
once between adjacent doubles -- and the Gauss-Legendre verifier accepts
them (reference tests/test_tables.py strategy)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def mods():
    from paper_1403_6870_b200 import construct, tables
    return construct, tables


def _ulps(a, b):
    return np.abs(a.view(np.int64) - b.view(np.int64))


@pytest.mark.parametrize("kind", ["exponential", "halfnormal"])
def test_build_reproduces_shipped_tables(mods, kind):
    construct, tables = mods
    built = construct.build_tables(kind, 256)
    shipped = tables.default_tables(kind)
    assert built.l_max == shipped.l_max and built.i_max == 256
    assert np.array_equal(built.f, shipped.f)           # layer heights: identical
    d = _ulps(built.x[1:], shipped.x[1:])
    assert (d != 0).sum() <= 2 and d.max() <= 8          # edges: at most 2 layers off by <= 8 ulp
    assert np.max(np.abs(built.a - shipped.a)) <= 1e-13 * shipped.a.max()
    assert abs(built.epsilon_max - shipped.epsilon_max) <= 1e-14


@pytest.mark.parametrize("kind", ["exponential", "halfnormal"])
def test_verify_accepts_shipped_tables(mods, kind):
    construct, tables = mods
    assert construct.verify_tables(tables.default_tables(kind)) == []


@pytest.mark.parametrize("i_max", [64, 512])
def test_other_sizes_build_and_verify(mods, i_max):
    construct, _ = mods
    for kind in ("exponential", "halfnormal"):
        t = construct.build_tables(kind, i_max)
        assert t.i_max == i_max and t.l_max < i_max
        assert construct.verify_tables(t) == []


def test_bad_inputs(mods):
    construct, tables = mods
    with pytest.raises(ValueError):
        construct.build_tables("exponential", 100)
    with pytest.raises(ValueError):
        construct.build_tables("cauchy", 256)
    t = tables.default_tables("exponential")
    bad = tables.ZigguratTables(distribution=t.distribution, i_max=t.i_max, l_max=t.l_max,
                                total_mass=t.total_mass, x=t.x, f=t.f, a=t.a[::-1].copy(),
                                epsilon_max=t.epsilon_max)
    assert "stored slot masses disagree with quadrature" in construct.verify_tables(bad)
