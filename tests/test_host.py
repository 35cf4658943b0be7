"""Host logic that needs no GPU: seeding, stream bookkeeping, statistics math,
path-count semantics, error surfaces."""
import math

import numpy as np
import pytest

import paper_1403_6870_b200 as zf
from paper_1403_6870_b200 import quality, uniform


def test_xoshiro_seeding_matches_reference_rule(orc):
    # four successive splitmix64 outputs of the seed (uniform.py:93-98)
    for seed in (0, 1, 42, 12345, 2**64 - 1):
        assert np.array_equal(uniform.xoshiro_seed_state(seed), orc.xoshiro_state(seed))
    assert np.array_equal(zf.UniformSource(1 << 64).state, zf.UniformSource(0).state)


def test_derive_seed(golden):
    for key, want in golden["derive_seed"].items():
        b, s = (int(x) for x in key.split(":"))
        assert zf.derive_seed(b, s) == want


def test_generators_and_errors():
    assert zf.UniformSource(5, generator="splitmix64").state.tolist() == [5]
    c = zf.UniformSource(5, generator="ctr")
    assert c.state.tolist() == [5, 0] and c.gid == 3
    assert zf.UniformSource.counter(9, 1 << 40).state.tolist() == [9, 1 << 40]
    with pytest.raises(ValueError):
        zf.UniformSource(0, generator="lcg128")
    with pytest.raises(ValueError):
        zf.UniformSource(0, generator="replay")
    with pytest.raises(ValueError):
        zf.UniformSource.replay([])


def test_replay_host_stream_wraps():
    src = zf.UniformSource.replay([5, 10, 15])
    assert [src.next_u64() for _ in range(7)] == [5, 10, 15, 5, 10, 15, 5]
    assert src.state[0] == 7
    dup = src.clone()
    assert dup.next_u64() == src.next_u64() == 10


def test_jump_bookkeeping():
    s = zf.UniformSource(3, generator="splitmix64")
    s.jump(10)
    assert int(s.state[0]) == (3 + 10 * 0x9E3779B97F4A7C15) % 2**64
    c = zf.UniformSource.counter(3, 5)
    c.jump(7)
    assert int(c.state[1]) == 12


def test_env_seed(monkeypatch):
    monkeypatch.setenv(uniform.SEED_ENV_VAR, "31337")
    assert zf.auto_seed_value() == 31337
    assert zf.UniformSource().seed == 31337
    monkeypatch.delenv(uniform.SEED_ENV_VAR)
    assert len({zf.auto_seed_value() for _ in range(8)}) > 1


def test_split_index():
    assert zf.split_index(0x1234, 8) == (0x34, 0x1234)
    with pytest.raises(zf.BitBudgetExceeded):
        zf.split_index(0, 13)
    with pytest.raises(ValueError):
        zf.split_index(0, 0)


def test_path_counts():
    c = zf.PathCounts.from_array([100, 98, 1, 1, 0, 2])
    assert c.common_fraction == 0.98 and c.tail_fraction == 0.0
    assert c.band_eval_fraction == 0.5
    assert zf.PathCounts(0, 0, 0, 0, 0, 0).common_fraction == 0.0


def test_quality_report_and_moment_math():
    rep = quality.QualityReport("normal", 100, [0.0, 1.0, 0.0, 3.0, 0.0],
                                [0.0, 1.0, 0.0, 3.0, 0.0], [1.0] * 5)
    assert rep.passed and "PASS" in rep.format_text() and rep.to_dict()["pass"]
    bad = quality.QualityReport("exp", 100, [8.0, 2, 6, 24, 120], [1.0, 2, 6, 24, 120], [1.0] * 5)
    assert not bad.passed
    m, v, s, k = quality.central_moments_from_raw([0.0, 1.0, 0.0, 3.0])
    assert (m, v, s, k) == (0.0, 1.0, 0.0, 0.0)
    m, v, s, k = quality.central_moments_from_raw([1.0, 2.0, 6.0, 24.0])  # Exp(1)
    assert (m, v) == (1.0, 1.0) and s == pytest.approx(2.0) and k == pytest.approx(6.0)


def test_histogram_chi2_against_exact_expectations():
    n, lo, hi, nb = 10**7, -6.0, 6.0, 64
    edges = np.linspace(lo, hi, nb + 1)
    cdf = np.array([quality.normal_cdf(e) for e in edges])
    probs = np.concatenate([[cdf[0]], np.diff(cdf), [1 - cdf[-1]]])
    hist = np.round(probs * n).astype(np.int64)
    chi2, dof, z = quality.histogram_chi2(hist, n, lo, hi)
    assert chi2 < 1.0 and dof > 10
    skewed = hist.copy()
    skewed[nb // 2] += 50_000
    assert quality.histogram_chi2(skewed, n, lo, hi)[2] > 6


def test_binomial_check():
    ok, mean, sd = quality.binomial_check(39397, 2**36, 5.7330e-7)
    assert ok and mean == pytest.approx(39397.5, rel=1e-3)
    assert not quality.binomial_check(45000, 2**36, 5.7330e-7)[0]


def test_expected_moments_table():
    assert quality.EXPECTED_MOMENTS["exp"] == (1.0, 2.0, 6.0, 24.0, 120.0)
    assert quality._MOMENT_SD["normal"][1] == math.sqrt(2.0)


def test_samplers_require_cuda_device():
    with pytest.raises(ValueError):
        zf.ExpSampler(device="cpu")


# the reference's zigfast.__all__ (zigfast/__init__.py:46-88)
REFERENCE_ALL = [
    "ALGORITHMS", "AliasTable", "BenchReport", "BitBudgetExceeded", "CurvatureViolation",
    "DensitySpec", "EXPECTED_MOMENTS", "EXPONENTIAL", "EmptyWeights", "ExpSampler", "FormatError",
    "HALF_NORMAL", "InvalidSpec", "NonConvergence", "NormalSampler", "QuadratureFailure",
    "QualityReport", "TraditionalExpSampler", "TraditionalNormalSampler", "TraditionalTables",
    "UniformSource", "ZigfastError", "ZigguratTables", "auto_seed_value", "build_alias",
    "build_tables", "compute_epsilon", "default_tables", "derive_seed", "exponential", "get",
    "half_normal", "load", "overhang_areas", "run_bench", "run_quality", "save", "solve_layers",
    "solve_traditional", "split_index", "verify_tables", "__version__",
]


def test_top_level_names_match_reference():
    import paper_1403_6870_b200 as zf
    missing = [n for n in REFERENCE_ALL if not hasattr(zf, n)]
    assert not missing
    assert set(REFERENCE_ALL) <= set(zf.__all__)
    # as in the reference, exponential / half_normal / get are DensitySpec factories
    spec = zf.exponential()
    assert isinstance(spec, zf.DensitySpec) and spec.kind == zf.EXPONENTIAL
    assert zf.half_normal().kind == zf.HALF_NORMAL and zf.get("exponential").kind == zf.EXPONENTIAL
    assert issubclass(zf.InvalidSpec, zf.ZigfastError)
    assert zf.ALGORITHMS == ("modified", "traditional")
