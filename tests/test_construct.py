"""Table construction: the restated solver reproduces the
reference's shipped i_max = 256 fixtures bit for bit, and the verifier
accepts them (reference tests/test_tables.py strategy)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def mods():
    from paper_1403_6870_b200 import construct, tables
    return construct, tables


@pytest.mark.parametrize("kind", ["exponential", "halfnormal"])
def test_build_reproduces_shipped_tables(mods, kind):
    construct, tables = mods
    built = construct.build_tables(kind, 256)
    shipped = tables.default_tables(kind)
    assert built.l_max == shipped.l_max
    for f in ("x", "f", "a"):
        assert np.array_equal(getattr(built, f), getattr(shipped, f)), f
    assert built.epsilon_max == shipped.epsilon_max
    assert built == shipped


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
