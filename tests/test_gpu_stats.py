"""Validation reductions and the fused generate-and-reduce kernel (production mode)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zf(cuda):
    import paper_1403_6870_b200 as zf
    return zf


def test_buffer_stats_match_numpy(zf, cuda):
    import torch
    from paper_1403_6870_b200 import quality
    x = torch.randn(1_000_003, dtype=torch.float64, device=cuda) * 2.0
    sums, res = quality.buffer_sums(x, hist=(-6.0, 6.0, 1024), thresholds=(1.0, 3.0, 7.5),
                                    abs_thresh=True)
    h = x.cpu().numpy()
    for k in range(5):
        want = math.fsum((h ** (k + 1)).tolist())
        assert sums[k] == pytest.approx(want, rel=1e-9, abs=1e-6)
    counts, _ = np.histogram(h, bins=1024, range=(-6.0, 6.0))
    assert res.hist[0] == (h < -6.0).sum() and res.hist[-1] == (h >= 6.0).sum()
    # the device bins with (x - lo) * (nbins / width); allow a handful of edge ties
    assert np.abs(res.hist[1:-1] - counts).sum() <= 4
    assert res.thresh_counts == [int((np.abs(h) > t).sum()) for t in (1.0, 3.0, 7.5)]


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_fused_stats_equal_fill_then_reduce(zf, cuda, dist):
    """zf_fill_stats draws exactly the samples zf_fill would write."""
    from paper_1403_6870_b200 import quality
    cls = zf.ExpSampler if dist == "exp" else zf.NormalSampler
    n = 3_000_001
    a = cls(source=zf.UniformSource.counter(5, 100), device=cuda)
    sums_f, res_f = quality.device_sums(a, n, hist=(-6.0, 6.0, 512), thresholds=(2.0, 4.0))
    b = cls(source=zf.UniformSource.counter(5, 100), device=cuda)
    x = b.fill(n)
    sums_b, res_b = quality.buffer_sums(x, hist=(-6.0, 6.0, 512), thresholds=(2.0, 4.0))
    assert np.array_equal(res_f.hist, res_b.hist)
    assert res_f.thresh_counts == res_b.thresh_counts
    for k in range(5):
        assert sums_f[k] == pytest.approx(sums_b[k], rel=1e-12, abs=1e-9)
    assert int(a.source.state[1]) == 100 + n


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_run_quality_passes(zf, cuda, dist):
    rep = zf.run_quality(dist, 1 << 24, seed=1234, device=cuda)
    assert rep.passed, rep.format_text()
    rep2 = zf.run_quality(dist, 1 << 20, seed=7, generator="xoshiro256++", device=cuda)
    assert rep2.passed, rep2.format_text()


@pytest.mark.parametrize("dist", ["normal", "exp"])
def test_run_quality_matches_reference(zf, golden, cuda, dist):
    """run_quality(dist, n, seed=7, jobs, chunk) (quality.py:109-138): the same
    xoshiro256++ shards (derive_seed) and chunking as the reference; moments
    equal the reference's up to the per-chunk summation order."""
    from helpers import hex_to_bits
    for key, want in golden["run_quality_seed7"].items():
        d, n, jobs, chunk = key.split(":")
        if d != dist:
            continue
        rep = zf.run_quality(dist, int(n), seed=7, jobs=int(jobs), chunk=int(chunk), device=cuda)
        ref = hex_to_bits(want["moments"]).view(np.float64)
        for k in range(5):
            assert rep.moments[k] == pytest.approx(ref[k], rel=1e-12, abs=1e-15), (key, k)
        assert rep.passed == want["passed"]


def test_tail_only_counts_equal_full_statistics(zf, cuda):
    """moments=0 with thresholds above every fast-path value counts on the rare
    path only (zf_stats_cfg.moments = 0); the counts equal the full
    statistics kernel's on the same stream (config-5 thresholds)."""
    from paper_1403_6870_b200 import quality
    x1 = float(zf.default_tables("exponential").x[1])
    n = 1 << 26
    for cls, th, ab in ((zf.NormalSampler, (5.0, 6.0, 4.0, 3.7), True),
                        (zf.ExpSampler, (x1, 9.0, 12.0), False)):
        a = cls(source=zf.UniformSource.counter(99, 1 << 40), device=cuda)
        _, fast = quality.device_sums(a, n, moments=0, thresholds=th, abs_thresh=ab)
        b = cls(source=zf.UniformSource.counter(99, 1 << 40), device=cuda)
        _, full = quality.device_sums(b, n, moments=5, thresholds=th, abs_thresh=ab)
        assert fast.thresh_counts == full.thresh_counts
        assert fast.thresh_counts[0] > 0
    # a threshold below the fast-path maximum falls back to the per-sample kernel
    c = zf.NormalSampler(source=zf.UniformSource.counter(1), device=cuda)
    _, r1 = quality.device_sums(c, 1 << 22, moments=0, thresholds=(2.0,), abs_thresh=True)
    d = zf.NormalSampler(source=zf.UniformSource.counter(1), device=cuda)
    _, r2 = quality.device_sums(d, 1 << 22, moments=5, thresholds=(2.0,), abs_thresh=True)
    assert r1.thresh_counts == r2.thresh_counts and r1.thresh_counts[0] > 100_000


def test_aggregate(zf, orc, golden, cuda):
    from helpers import hex_to_bits
    for dist, cls in (("exp", zf.ExpSampler), ("normal", zf.NormalSampler)):
        s = cls(source=zf.UniformSource(11), device=cuda)
        got = s.aggregate(20000)
        want = hex_to_bits([golden[f"{dist}_seed11_aggregate20000"]]).view(np.float64)[0]
        # the reference sums left to right; ours is an exact merge of block sums
        assert got == pytest.approx(want, rel=1e-12, abs=1e-9)
        p = cls(source=zf.UniformSource.counter(3), device=cuda)
        vals, _, _ = orc.fill_ctr(dist, 1_000_000, seed=3)
        assert p.aggregate(1_000_000) == pytest.approx(math.fsum(vals.tolist()), rel=1e-12)


def test_config2_validation(zf, cuda):
    """BASELINE config 2: N(0,1), n = 2^28, seed 1234: mean/var/skew/kurtosis
    within 6 sigma and the 1024-bin histogram on [-6, 6] vs the analytic CDF."""
    from paper_1403_6870_b200 import quality
    n = 1 << 28
    s = zf.NormalSampler(source=zf.UniformSource.counter(1234), device=cuda)
    sums, res = quality.device_sums(s, n, hist=(-6.0, 6.0, 1024))
    mean, var, skew, exk = quality.central_moments_from_raw([v / n for v in sums])
    for val, se in ((mean, (1 / n) ** 0.5), (var - 1, (2 / n) ** 0.5), (skew, (6 / n) ** 0.5),
                    (exk, (24 / n) ** 0.5)):
        assert abs(val / se) < 6.0
    chi2, dof, z = quality.histogram_chi2(res.hist, n, -6.0, 6.0)
    assert abs(z) < 6.0, (chi2, dof)


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_tail_mass(zf, cuda, dist):
    """Tail counts vs analytic tail mass within a 5-sigma binomial bound (config 5 shape)."""
    from paper_1403_6870_b200 import quality
    n = 1 << 30
    if dist == "normal":
        s = zf.NormalSampler(source=zf.UniformSource.counter(99), device=cuda)
        _, res = quality.device_sums(s, n, thresholds=(3.0, 4.0, 5.0), abs_thresh=True)
        for t, c in zip((3.0, 4.0, 5.0), res.thresh_counts):
            ok, mean, sd = quality.binomial_check(c, n, math.erfc(t / math.sqrt(2.0)))
            assert ok, (t, c, mean, sd)
    else:
        x1 = zf.default_tables("exponential").x[1]
        s = zf.ExpSampler(source=zf.UniformSource.counter(99), device=cuda)
        _, res = quality.device_sums(s, n, thresholds=(1.0, x1, 10.0))
        for t, c in zip((1.0, x1, 10.0), res.thresh_counts):
            ok, mean, sd = quality.binomial_check(c, n, math.exp(-t))
            assert ok, (t, c, mean, sd)
