"""Scale configurations across ranks (BASELINE.json configs 3 and 5).

One process per GPU; rank r owns counter range [r * 2^40, ...) of the seed
(`shard.counter_base`), so no samples cross ranks and the only collective is a
SUM allreduce of validation statistics (NCCL on GPUs, gloo in the CPU tests).
The reference's analogue is `run_quality`'s per-job samplers seeded
`derive_seed(base, i)` merged with `math.fsum` (quality.py:118-129).

The statistics calls are injectable (`stats=`) so the multi-rank host logic --
shares, counter bases, packing, the allreduce and the final checks -- is
exercised at world size 2 over gloo with the CPU oracle standing in for the
kernels (tests/test_multiproc.py); bench.py runs the same functions with the
device kernels over NCCL.
"""

from __future__ import annotations

import math

from . import quality, shard

C3_SEED = 7
C3_HIST = (-6.0, 6.0, 1024)
C3_THRESH = (5.0, 6.0, 7.0)
C5_SEED = 99
C5_THRESH = (5.0, 6.0, 7.0)


def share(total: int, rank: int, world: int) -> int:
    """Rank's share of ``total`` samples (the reference's job split,
    quality.py:122)."""
    if not 0 <= rank < world:
        raise ValueError("rank outside the world")
    return total // world + (1 if rank < total % world else 0)


# -- device statistics (the default `stats` implementations) --------------------

def device_counts(dist: str, seed: int, ctr_base: int, n: int, thresholds, abs_thresh: bool,
                  device=None) -> list[int]:
    """Generate-and-count on the device: ``n`` draws of the counter stream
    (seed, ctr_base), counts of x > t (|x| > t), nothing stored (fused
    statistics kernel, tail-only mode when every threshold is above the
    fast path)."""
    from .samplers import ExpSampler, NormalSampler
    from .uniform import UniformSource
    cls = NormalSampler if dist == "normal" else ExpSampler
    s = cls(source=UniformSource.counter(seed, ctr_base), device=device)
    _, res = quality.device_sums(s, n, moments=0, thresholds=tuple(thresholds),
                                 abs_thresh=abs_thresh)
    return list(res.thresh_counts)


def buffer_stats(x, hist=C3_HIST, thresholds=C3_THRESH):
    """Moment sums, histogram and |x| tail counts of a device buffer."""
    sums, res = quality.buffer_sums(x, hist=hist, thresholds=thresholds, abs_thresh=True)
    return list(sums), [int(v) for v in res.hist.tolist()], list(res.thresh_counts)


# -- config 3: validation of the per-rank fills ---------------------------------

def validate_config3(sums, hist, tails, n_local: int, device=None,
                     lo: float = C3_HIST[0], hi: float = C3_HIST[1],
                     thresholds=C3_THRESH) -> dict:
    """Reduce every rank's statistics (one SUM allreduce of ~1 k numbers) and
    check the union against N(0,1): central moments with z-scores, the
    1024-bin chi-square against the analytic CDF, |x| > 5, 6, 7 against the
    binomial tail mass.  Every rank returns the same report."""
    vec = shard.allreduce_stats([float(n_local)] + shard.pack_stats(sums, hist, tails),
                                device=device)
    tot = int(round(vec[0]))
    rs, rh, rt = shard.unpack_stats(vec[1:], len(sums), len(hist), len(tails))
    mean, var, skew, exkurt = quality.central_moments_from_raw([s / tot for s in rs[:4]])
    import numpy as np
    chi2, dof, chi2_z = quality.histogram_chi2(np.array(rh), tot, lo, hi)
    tail_rows = []
    for t, c in zip(thresholds, rt):
        ok, m, sd = quality.binomial_check(int(c), tot, math.erfc(t / math.sqrt(2.0)))
        tail_rows.append({"abs_gt": t, "count": int(c), "expected": m, "sd": sd,
                          "within_5sigma": ok})
    z = [mean / math.sqrt(1 / tot), (var - 1) / math.sqrt(2 / tot), skew / math.sqrt(6 / tot),
         exkurt / math.sqrt(24 / tot)]
    return {"n_total": tot, "mean": mean, "var": var, "skew": skew, "excess_kurtosis": exkurt,
            "z": z, "hist_chi2": chi2, "hist_dof": dof, "hist_z": chi2_z, "tails": tail_rows,
            "passed": all(abs(v) <= 6.0 for v in z) and abs(chi2_z) <= 6.0
            and all(r["within_5sigma"] for r in tail_rows)}


# -- config 5: tail stress --------------------------------------------------------

def config5(total: int, rank: int, world: int, device=None, seed: int = C5_SEED,
            stats=None, exp_x1: float | None = None) -> dict:
    """Rank's share of ``total`` N(0,1) and ``total`` Exp(1) draws, generated
    and counted in the kernel (|x| > 5, 6, 7 and x > X[1]), then one SUM
    allreduce of the 4 counts.  Every rank returns the same report."""
    stats = stats or (lambda *a: device_counts(*a, device=device))
    if exp_x1 is None:
        from .tables import default_tables
        exp_x1 = float(default_tables("exponential").x[1])
    m = share(total, rank, world)
    base = shard.counter_base(rank)
    cn = stats("normal", seed, base, m, C5_THRESH, True)
    ce = stats("exp", seed, base, m, (exp_x1,), False)
    red = shard.allreduce_stats([float(c) for c in list(cn) + list(ce)], device=device)
    counts = [int(round(v)) for v in red]
    rows = []
    for t, c in zip(C5_THRESH, counts[:3]):
        ok, mean, sd = quality.binomial_check(c, total, math.erfc(t / math.sqrt(2.0)))
        rows.append({"abs_gt": t, "count": c, "expected": mean, "sd": sd, "within_5sigma": ok})
    ok, mean, sd = quality.binomial_check(counts[3], total, math.exp(-exp_x1))
    return {"n_total_per_dist": total, "share": m, "normal_abs_tails": rows,
            "exp_beyond_X1": {"X1": exp_x1, "count": counts[3], "expected": mean, "sd": sd,
                              "within_5sigma": ok},
            "passed": ok and all(r["within_5sigma"] for r in rows)}
