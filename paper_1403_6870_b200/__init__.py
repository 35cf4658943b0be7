"""paper_1403_6870_b200 -- modified-ziggurat Exponential(1) / N(0,1) sampling on B200.

A B200-native (sm_100a) re-build of the sampling path of the reference package
`zigfast` (McFarland, arXiv 1403.6870): the same top-level names as the
reference's `zigfast/__init__.py:9-88` (samplers, sources, tables, alias,
densities, errors, quality, bench harness), with every draw computed by
hand-written CUDA kernels behind a C-ABI (include/zigfast_b200.h).

As in the reference, `exponential()` / `half_normal()` / `get()` are the
DensitySpec factories.  The convenience draw functions -- `seed(v)`,
`standard_exponential(size)` and `standard_normal(size)` (alias `normal`, the
SPEC name from the reference's TS frontend, free because the reference has no
top-level `normal`) -- draw from the production counter stream of one
module-level seed.
"""

from __future__ import annotations

import threading

from .errors import (BitBudgetExceeded, CurvatureViolation, DeviceError, EmptyWeights,
                     ExtensionMissing, FormatError, InvalidSpec, NonConvergence,
                     QuadratureFailure, ZigfastError)
from .batch import BatchPlan, fill_batch
from .bench import ALGORITHMS, BenchReport, run_bench
from .construct import (DensitySpec, build_tables, compute_epsilon, exponential, get,
                        half_normal, overhang_areas, solve_layers, verify_tables)
from .quality import EXPECTED_MOMENTS, QualityReport, run_quality
from .samplers import ExpSampler, NormalSampler, PathCounts
from .tables import (EXPONENTIAL, HALF_NORMAL, AliasTable, ZigguratTables, build_alias,
                     default_tables, load, save)
from .traditional import (TraditionalExpSampler, TraditionalNormalSampler, TraditionalTables,
                          solve_traditional)
from .uniform import UniformSource, auto_seed_value, derive_seed, split_index

__version__ = "0.1.0"

_conv_lock = threading.Lock()
_conv = {"seed": None, "counter": 0}


def seed(value: int | None = None) -> int:
    """(Re)seed the convenience stream; returns the seed in use."""
    with _conv_lock:
        _conv["seed"] = (auto_seed_value() if value is None else int(value)) & ((1 << 64) - 1)
        _conv["counter"] = 0
        return _conv["seed"]


def _convenience(dist_cls, size: int, device=None):
    with _conv_lock:
        if _conv["seed"] is None:
            _conv["seed"] = auto_seed_value()
        src = UniformSource.counter(_conv["seed"], _conv["counter"])
        _conv["counter"] += int(size)
    return dist_cls(source=src, device=device).fill(int(size))


def standard_exponential(size: int, device=None):
    """``size`` Exponential(1) draws (CUDA float64 tensor), continuing the stream."""
    return _convenience(ExpSampler, size, device)


def standard_normal(size: int, device=None):
    """``size`` N(0,1) draws (CUDA float64 tensor), continuing the stream."""
    return _convenience(NormalSampler, size, device)


normal = standard_normal


__all__ = [
    # the reference's zigfast.__all__ (zigfast/__init__.py:46-88)
    "ALGORITHMS", "AliasTable", "BenchReport", "BitBudgetExceeded", "CurvatureViolation",
    "DensitySpec", "EXPECTED_MOMENTS", "EXPONENTIAL", "EmptyWeights", "ExpSampler", "FormatError",
    "HALF_NORMAL", "InvalidSpec", "NonConvergence", "NormalSampler", "QuadratureFailure",
    "QualityReport", "TraditionalExpSampler", "TraditionalNormalSampler", "TraditionalTables",
    "UniformSource", "ZigfastError", "ZigguratTables", "auto_seed_value", "build_alias",
    "build_tables", "compute_epsilon", "default_tables", "derive_seed", "exponential", "get",
    "half_normal", "load", "overhang_areas", "run_bench", "run_quality", "save", "solve_layers",
    "solve_traditional", "split_index", "verify_tables", "__version__",
    # B200 additions
    "BatchPlan", "DeviceError", "ExtensionMissing", "PathCounts", "fill_batch", "normal", "seed",
    "standard_exponential", "standard_normal",
]
