"""Production-mode validation: moments, histogram and tail-mass checks.

Mirrors `zigfast/quality.py` (raw moments k=1..5 with analytic standard
errors, |z| <= 6 gate, `QualityReport`) and adds the checks BASELINE.json asks
for at scale: central moments, a 1024-bin histogram on [-6, 6] against the
analytic CDF (chi-square), and tail counts against binomial bounds.

All reductions run on the device (`zf_fill_stats` fuses generation and
reduction without writing samples; `zf_stats` reduces an existing buffer).
Partial sums come back per block and are merged with `math.fsum`, exactly as
the reference merges its per-chunk sums (`quality.py:129`).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

EXPECTED_MOMENTS = {
    "exp": (1.0, 2.0, 6.0, 24.0, 120.0),
    "normal": (0.0, 1.0, 0.0, 3.0, 0.0),
}
_MOMENT_SD = {
    "exp": tuple(math.sqrt(math.factorial(2 * k) - math.factorial(k) ** 2) for k in range(1, 6)),
    "normal": (1.0, math.sqrt(2.0), math.sqrt(15.0), math.sqrt(96.0), math.sqrt(945.0)),
}


@dataclass
class StatsResult:
    n: int
    sums: list            # fsum-merged sum of x^k, k = 1..5
    hist: np.ndarray      # [under, bins..., over] (empty if disabled)
    thresh_counts: list   # per threshold
    thresholds: list

    def raw_moments(self):
        return [s / self.n for s in self.sums]


def _cfg(hist=None, thresholds=(), abs_thresh=False, moments=5) -> _lib.StatsCfg:
    if not 0 <= moments <= 5:
        raise ValueError("moments must be in 0..5")
    if moments == 0 and hist is None and not thresholds:
        raise ValueError("nothing to compute: no moments, histogram or thresholds")
    cfg = _lib.StatsCfg()
    # 1 moment with no histogram / thresholds selects the sum-only kernel; 0
    # moments with thresholds above every fast-path value the rare-path-only
    # tail counter (zigfast_b200.h, zf_stats_cfg.moments)
    cfg.moments = moments if moments <= 1 else 5
    if hist is not None:
        cfg.hist_lo, cfg.hist_hi, cfg.nbins = float(hist[0]), float(hist[1]), int(hist[2])
    if len(thresholds) > 8:
        raise ValueError("at most 8 thresholds")
    cfg.nthresh = len(thresholds)
    cfg.abs_thresh = int(abs_thresh)
    for i, t in enumerate(thresholds):
        cfg.thresh[i] = float(t)
    return cfg


def _collect(n, partials, counts, cfg, thresholds, moments: int = 5) -> StatsResult:
    p = partials.cpu().numpy().reshape(-1, 5)
    c = counts.cpu().numpy().astype(np.int64) if (cfg.nbins or cfg.nthresh) else None
    # exact merge of the per-block rows; unrequested moments are not summed
    sums = [math.fsum(p[:, k].tolist()) if k < moments else math.nan for k in range(5)]
    if c is None:
        return StatsResult(n=n, sums=sums, hist=np.zeros(0, dtype=np.int64), thresh_counts=[],
                           thresholds=list(thresholds))
    nb = cfg.nbins
    hist = c[:nb + 2] if nb else np.zeros(0, dtype=np.int64)
    # counts layout: [nbins + 2 histogram slots][thresholds] (2 unused slots if nbins == 0)
    tc = [int(v) for v in c[nb + 2:nb + 2 + cfg.nthresh]]
    return StatsResult(n=n, sums=sums, hist=hist, thresh_counts=tc, thresholds=list(thresholds))


def _buffers(device, n, cfg):
    import torch
    blocks = _lib.lib().zf_stats_blocks(n)
    partials = torch.zeros(blocks * 5, dtype=torch.float64, device=device)
    ncounts = (cfg.nbins + 2 if cfg.nbins else 2) + 8
    counts = torch.zeros(ncounts, dtype=torch.int64, device=device)
    return partials, counts


def device_sums(sampler, n: int, moments: int = 5, hist=None, thresholds=(), abs_thresh=False):
    """Generate ``n`` draws from a production sampler and reduce them on the
    fly (no HBM writes); advances the sampler's counter.  Returns
    (sums[:moments], StatsResult)."""
    import torch
    src = sampler.source
    if src.gid != _lib.GEN_CTR:
        raise ValueError("fused statistics need a production ('ctr') source")
    cfg = _cfg(hist, thresholds, abs_thresh, moments)
    partials, counts = _buffers(sampler.device, n, cfg)
    with torch.cuda.device(sampler.device):
        _lib.check(_lib.lib().zf_fill_stats(
            sampler._dev_tables.handle, sampler._dist, int(src.state[0]), int(src.state[1]), n,
            C.byref(cfg), partials.data_ptr(), counts.data_ptr(),
            _lib.stream_handle(sampler.device)))
    src.state[1] = np.uint64(int(src.state[1]) + n)
    res = _collect(n, partials, counts, cfg, thresholds, moments)
    return res.sums[:moments], res


def buffer_sums(x, moments: int = 5, hist=None, thresholds=(), abs_thresh=False):
    """Reduce an existing CUDA tensor (float64/float32)."""
    import torch
    cfg = _cfg(hist, thresholds, abs_thresh)
    n = x.numel()
    partials, counts = _buffers(x.device, n, cfg)
    dtype = _lib.F64 if x.dtype == torch.float64 else _lib.F32
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().zf_stats(dtype, x.data_ptr(), n, C.byref(cfg), partials.data_ptr(),
                                       counts.data_ptr(), _lib.stream_handle(x.device)))
    res = _collect(n, partials, counts, cfg, thresholds, moments)
    return res.sums[:moments], res


# ---------------------------------------------------------------------------
# reference-compatible report
# ---------------------------------------------------------------------------

@dataclass
class QualityReport:
    distribution: str
    n: int
    moments: list
    expected: list
    standard_errors: list
    z_scores: list = field(init=False)
    passed: bool = field(init=False)

    def __post_init__(self):
        self.z_scores = [(m - e) / se for m, e, se in
                         zip(self.moments, self.expected, self.standard_errors)]
        self.passed = all(abs(z) <= 6.0 for z in self.z_scores)

    def to_dict(self) -> dict:
        return {"distribution": self.distribution, "n": self.n, "moments": self.moments,
                "expected": self.expected, "standard_errors": self.standard_errors,
                "z_scores": self.z_scores, "pass": self.passed}

    def format_text(self) -> str:
        lines = [f"Created {self.n} {self.distribution} distributed pseudo-random numbers..."]
        for k, (m, z) in enumerate(zip(self.moments, self.z_scores), start=1):
            lines.append(f"X{k}: {m:.6f}  (z = {z:+.2f})")
        lines.append("PASS" if self.passed else "FAIL")
        return "\n".join(lines)


def make_sampler(dist: str, seed, generator: str = "xoshiro256++", device=None):
    """`quality.make_sampler` (quality.py:83-89); ``generator`` defaults to the
    reference's own stream, "ctr" selects the production counter stream."""
    from .samplers import ExpSampler, NormalSampler
    from .uniform import UniformSource
    source = UniformSource(seed, generator=generator)
    if dist == "exp":
        return ExpSampler(source=source, device=device)
    if dist == "normal":
        return NormalSampler(source=source, device=device)
    raise ValueError(f"unknown distribution: {dist!r}")


def _moment_sums(sampler, n: int, chunk: int) -> list[list[float]]:
    """Per-chunk power sums of ``n`` draws (quality.py:92-106): the sampler
    fills one reused device chunk at a time, exactly as the reference fills
    views of one host buffer, so the stream is consumed identically; each
    chunk is reduced on the device."""
    import torch
    sums: list[list[float]] = [[] for _ in range(5)]
    if sampler.source.gid == _lib.GEN_CTR:  # production: fused, nothing stored
        s, _ = device_sums(sampler, n)
        for k in range(5):
            sums[k].append(s[k])
        return sums
    buf = torch.empty(min(chunk, n), dtype=torch.float64, device=sampler.device)
    left = n
    while left > 0:
        m = min(chunk, left)
        view = buf[:m]
        sampler.fill(view)
        s, _ = buffer_sums(view)
        for k in range(5):
            sums[k].append(s[k])
        left -= m
    return sums


def run_quality(dist: str, n: int, seed=None, jobs: int = 1, chunk: int = 1 << 22,
                generator: str = "xoshiro256++", device=None) -> QualityReport:
    """First five raw moments of ``n`` draws vs their analytic values
    (`quality.py:109-138`): ``jobs`` shards seeded ``derive_seed(base, i)``
    with the reference's share split, every shard consuming its stream as the
    reference does, per-chunk sums merged with ``math.fsum``.  The shards run
    one after another (each fill already spans every SM).  The draws are the
    reference's bit for bit; the per-chunk sums are fsum-exact rather than
    numpy's pairwise order (|difference| ~1e-16 relative per chunk)."""
    from .uniform import UniformSource, derive_seed
    if dist not in EXPECTED_MOMENTS:
        raise ValueError(f"unknown distribution: {dist!r}")
    if n <= 0:
        raise ValueError("n must be positive")
    jobs = max(1, jobs)
    if jobs == 1:
        all_sums = _moment_sums(make_sampler(dist, seed, generator, device), n, chunk)
    else:
        base = seed if seed is not None else UniformSource().seed
        shares = [n // jobs + (1 if i < n % jobs else 0) for i in range(jobs)]
        parts = [_moment_sums(make_sampler(dist, derive_seed(base, i), generator, device), m,
                              chunk)
                 for i, m in enumerate(shares) if m > 0]
        all_sums = [[s for part in parts for s in part[k]] for k in range(5)]
    moments = [math.fsum(all_sums[k]) / n for k in range(5)]
    ses = [sd / math.sqrt(n) for sd in _MOMENT_SD[dist]]
    return QualityReport(distribution=dist, n=n, moments=moments,
                         expected=list(EXPECTED_MOMENTS[dist]), standard_errors=ses)


# ---------------------------------------------------------------------------
# scale checks (BASELINE.json configs 2, 3, 5)
# ---------------------------------------------------------------------------

def normal_cdf(x):
    return 0.5 * math.erfc(-x / math.sqrt(2.0))


def central_moments_from_raw(raw):
    """mean, variance, skewness, excess kurtosis from raw moments E[x^1..4]."""
    m1, m2, m3, m4 = raw[:4]
    var = m2 - m1 * m1
    mu3 = m3 - 3 * m1 * m2 + 2 * m1 ** 3
    mu4 = m4 - 4 * m1 * m3 + 6 * m1 * m1 * m2 - 3 * m1 ** 4
    return m1, var, mu3 / var ** 1.5, mu4 / var ** 2 - 3.0


def histogram_chi2(hist: np.ndarray, n: int, lo: float, hi: float, cdf=normal_cdf):
    """Pearson chi-square of [under, bins..., over] against a CDF; returns
    (chi2, dof, z) with z = (chi2 - dof)/sqrt(2 dof).  Bins with expectation
    below 5 are pooled with their neighbour."""
    nb = hist.size - 2
    edges = np.linspace(lo, hi, nb + 1)
    cdfv = np.array([cdf(e) for e in edges])
    probs = np.concatenate([[cdfv[0]], np.diff(cdfv), [1.0 - cdfv[-1]]])
    exp = probs * n
    obs = hist.astype(np.float64)
    # pool small-expectation cells left to right
    po, pe, acc_o, acc_e = [], [], 0.0, 0.0
    for o, e in zip(obs, exp):
        acc_o += o
        acc_e += e
        if acc_e >= 5.0:
            po.append(acc_o)
            pe.append(acc_e)
            acc_o = acc_e = 0.0
    if acc_e > 0 and pe:
        po[-1] += acc_o
        pe[-1] += acc_e
    po, pe = np.array(po), np.array(pe)
    chi2 = float(((po - pe) ** 2 / pe).sum())
    dof = len(pe) - 1
    return chi2, dof, (chi2 - dof) / math.sqrt(2 * dof)


def binomial_check(count: int, n: int, p: float, sigmas: float = 5.0):
    """Whether ``count`` is within ``sigmas`` binomial SDs of n*p (+1 for tiny means)."""
    mean = n * p
    sd = math.sqrt(n * p * (1 - p))
    return abs(count - mean) <= sigmas * sd + 1.0, mean, sd
