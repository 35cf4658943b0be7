"""Generate-and-aggregate benchmark harness on the device (`zigfast/bench.py`).

Same API as the reference: ``run_bench(algorithms, dist, n, trials, seed)``
times ``sampler.aggregate(n)`` (draws summed without being stored, so nothing
can be skipped) for the modified and the traditional ziggurat, reports the
median of >= 3 trials and the modified algorithm's speed-up over the
traditional one (the reference's acceptance criterion 6 asks for >= 1.2x).
``generator`` picks the stream: the reference's xoshiro256++ (oracle mode,
default, as in the reference) or ``"ctr"`` (production).
"""

from __future__ import annotations

import statistics
import time
from dataclasses import dataclass, field

from .samplers import ExpSampler, NormalSampler
from .traditional import TraditionalExpSampler, TraditionalNormalSampler
from .uniform import UniformSource

ALGORITHMS = ("modified", "traditional")


@dataclass
class BenchReport:
    algorithm: str
    distribution: str
    n: int
    trials: int
    median_seconds: float
    throughput: float = field(init=False)
    speedup_vs_baseline: float | None = None
    trial_seconds: list = field(default_factory=list)

    def __post_init__(self):
        self.throughput = self.n / self.median_seconds if self.median_seconds else 0.0

    def to_dict(self) -> dict:
        return {"algorithm": self.algorithm, "distribution": self.distribution, "n": self.n,
                "trials": self.trials, "median_seconds": self.median_seconds,
                "throughput": self.throughput, "speedup_vs_baseline": self.speedup_vs_baseline,
                "trial_seconds": self.trial_seconds}


def _make(algorithm: str, dist: str, seed, generator: str, device):
    src = (UniformSource.counter(seed) if generator == "ctr"
           else UniformSource(seed, generator=generator))
    table = {("modified", "exp"): ExpSampler, ("modified", "normal"): NormalSampler,
             ("traditional", "exp"): TraditionalExpSampler,
             ("traditional", "normal"): TraditionalNormalSampler}
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm: {algorithm!r}")
    return table[(algorithm, dist)](source=src, device=device)


def run_bench(algorithms, dist: str, n: int, trials: int = 3, seed: int | None = None,
              generator: str = "xoshiro256++", device=None) -> list[BenchReport]:
    """Time each algorithm's aggregate(n); median of ``trials`` (>= 3)."""
    if dist not in ("exp", "normal"):
        raise ValueError(f"unknown distribution: {dist!r}")
    if trials < 3:
        raise ValueError("need at least 3 trials for a stable median")
    reports = []
    for algorithm in algorithms:
        sampler = _make(algorithm, dist, seed, generator, device)
        sampler.aggregate(1000)  # tables upload, kernel load
        times = []
        for _ in range(trials):
            t0 = time.perf_counter()
            sampler.aggregate(n)  # returns a host float: synchronised
            times.append(time.perf_counter() - t0)
        reports.append(BenchReport(algorithm=algorithm, distribution=dist, n=n, trials=trials,
                                   median_seconds=statistics.median(times), trial_seconds=times))
    by_name = {r.algorithm: r for r in reports}
    if "modified" in by_name and "traditional" in by_name:
        by_name["modified"].speedup_vs_baseline = (by_name["traditional"].median_seconds /
                                                   by_name["modified"].median_seconds)
    return reports
