"""Traditional ziggurat baseline, CPU side: the oracle and the product's table
solver against the reference (golden fixtures from tests/golden/make_golden.py
and the reference's own golden draws, tests/test_traditional.py:15-29)."""
import hashlib

import numpy as np
import pytest

from helpers import assert_bits_equal, bits, hex_to_bits

TRAD = ["trad_exp", "trad_normal"]
KIND = {"trad_exp": "exponential", "trad_normal": "halfnormal"}

# reference tests/test_traditional.py:15-29
GOLDEN_EXP_SEED7 = [0.15251242197550072, 0.72345693135302247, 1.3292620703893605,
                    1.1865778989015741, 1.7335432749258897]
GOLDEN_NORMAL_SEED7 = [0.22743262333957229, 0.89875818955456432, -0.9216075305818846,
                       1.7633235223206458, -0.11656456605859367]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def check_tables(g, x, f, k, r, v, se, kk, flo, fh):
    assert bits([r])[0] == int(g["r"], 16)
    assert bits([v])[0] == int(g["v"], 16)
    assert sha(x) == g["x_sha256"] and sha(f) == g["f_sha256"] and sha(k) == g["k_sha256"]
    assert sha(se) == g["se_sha256"] and sha(np.asarray(kk, np.uint64)) == g["kk_sha256"]
    assert sha(flo) == g["flo_sha256"] and sha(fh) == g["fh_sha256"]


@pytest.mark.parametrize("dist", TRAD)
def test_oracle_tables_match_reference(orc, golden, dist):
    p = orc.OracleTradPack(KIND[dist])
    check_tables(golden[f"{dist}_tables"], p.x, p.f, p.k, p.r, p.v, p.se, p.kk, p.flo, p.fh)


@pytest.mark.parametrize("dist", TRAD)
def test_product_solver_matches_reference(golden, dist):
    from paper_1403_6870_b200 import traditional as T
    t = T.solve_traditional(KIND[dist], 256)
    p = T.trad_pack(t)
    check_tables(golden[f"{dist}_tables"], t.x, t.f, t.k, t.r, t.v, p.se, p.kk, p.flo, p.fh)
    assert t.fast_accept_probability() == golden[f"{dist}_tables"]["fast_accept_probability"]


@pytest.mark.parametrize("kind", ["exponential", "halfnormal"])
def test_stack_properties(kind):
    """traditional.py invariants (reference tests/test_traditional.py:32-57)."""
    from paper_1403_6870_b200 import traditional as T
    t = T.solve_traditional(kind, 256)
    assert t.f[-1] == 1.0 and t.x[-1] == 0.0
    assert np.all(np.diff(t.x) < 0.0) and np.all(np.diff(t.f) > 0.0)
    strips = t.x[:-1] * np.diff(t.f)
    np.testing.assert_allclose(strips, t.v, rtol=1e-9)
    assert np.all(t.k[:-1] > 0.0) and np.all(t.k <= 1.0) and t.k[-1] == 0.0
    assert 0.97 < t.fast_accept_probability() < 0.99
    assert t.edge[0] == t.v / t.f[0]
    np.testing.assert_array_equal(t.edge[1:], t.x[:-1])
    with pytest.raises(ValueError):
        T.solve_traditional(kind, 100)


def test_oracle_golden_first_draws(orc):
    assert list(orc.fill_stream("trad_exp", 5, seed=7)[0]) == GOLDEN_EXP_SEED7
    assert list(orc.fill_stream("trad_normal", 5, seed=7)[0]) == GOLDEN_NORMAL_SEED7


@pytest.mark.parametrize("dist", TRAD)
def test_oracle_fills_counts_aggregate(orc, golden, dist):
    assert_bits_equal(orc.fill_stream(dist, 3000, seed=7)[0],
                      hex_to_bits(golden[f"{dist}_seed7_fill3000"]), "seed 7")
    assert_bits_equal(orc.fill_stream(dist, 2000, generator="splitmix64", seed=99)[0],
                      hex_to_bits(golden[f"{dist}_splitmix99_fill2000"]), "splitmix 99")
    _, cnt, _, _ = orc.fill_stream(dist, 200_000, seed=3)
    assert cnt.tolist() == golden[f"{dist}_seed3_counts200k"]
    agg = orc.aggregate(dist, 20000, 11)
    assert bits([agg])[0] == int(golden[f"{dist}_seed11_aggregate20000"], 16)


@pytest.mark.parametrize("dist", TRAD)
def test_oracle_replay_kats(orc, golden, dist):
    for label, kat in golden[f"{dist}_kat"].items():
        w = [int(h, 16) for h in kat["words"]]
        v, _, _, used = orc.fill_stream(dist, 1, replay_words=w)
        assert bits(v)[0] == int(kat["value"], 16), label
        assert used == kat["cursor"], label


@pytest.mark.parametrize("dist", TRAD)
def test_oracle_config1_records(orc, golden, dist):
    g = golden[f"c1_{dist}"]
    vals, cnt, recs, used = orc.fill_stream(dist, g["n"], seed=42, records=True)
    assert sha(vals) == g["values_sha256"]
    assert sha(recs["start"]) == g["starts_sha256"]
    assert sha(recs["nwords"]) == g["nwords_sha256"]
    assert sha(recs["layer"]) == g["layer_sha256"]
    assert sha(recs["path"]) == g["path_sha256"]
    if g["attempts_sha256"]:
        assert sha(recs["attempts"]) == g["attempts_sha256"]
    assert cnt.tolist() == g["counters"] and used == g["words_consumed"]


@pytest.mark.parametrize("dist", TRAD)
def test_oracle_production_stream_matches_reference_replay(orc, golden, dist):
    for key, want in golden[f"ctr_{dist}"].items():
        seed, base = (int(x) for x in key.split(":"))
        got, _, _ = orc.fill_ctr(dist, len(want), seed=seed, ctr_base=base)
        assert_bits_equal(got, hex_to_bits(want), key)
