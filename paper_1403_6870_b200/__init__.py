"""paper_1403_6870_b200 -- modified-ziggurat Exponential(1) / N(0,1) sampling on B200.

A B200-native (sm_100a) re-build of the sampling path of the reference package
`zigfast` (McFarland, arXiv 1403.6870): same Python API (`ExpSampler`,
`NormalSampler`, `UniformSource`, tables, alias, quality), with every draw
computed by hand-written CUDA kernels behind a C-ABI (include/zigfast_b200.h).

Convenience surface (SPEC `exponential(size)`, `normal(size)`, `seed(v)`,
realised in the reference only by its TS frontend) draws from the production
counter stream of one module-level seed.
"""

from __future__ import annotations

import threading

from .errors import (BitBudgetExceeded, DeviceError, EmptyWeights, ExtensionMissing,
                     FormatError, NonConvergence, ZigfastError)
from .batch import BatchPlan, fill_batch
from .construct import build_tables, verify_tables
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


def exponential(size: int, device=None):
    """``size`` Exponential(1) draws (CUDA float64 tensor), continuing the stream."""
    return _convenience(ExpSampler, size, device)


def normal(size: int, device=None):
    """``size`` N(0,1) draws (CUDA float64 tensor), continuing the stream."""
    return _convenience(NormalSampler, size, device)


__all__ = [
    "AliasTable", "BatchPlan", "build_tables", "verify_tables", "BitBudgetExceeded", "DeviceError", "EXPECTED_MOMENTS", "EXPONENTIAL",
    "EmptyWeights", "ExpSampler", "ExtensionMissing", "FormatError", "HALF_NORMAL",
    "NonConvergence", "NormalSampler", "PathCounts", "QualityReport",
    "TraditionalExpSampler", "TraditionalNormalSampler", "TraditionalTables", "UniformSource",
    "ZigfastError",
    "ZigguratTables", "auto_seed_value", "build_alias", "default_tables", "derive_seed",
    "exponential", "fill_batch", "load", "normal", "run_quality", "save", "seed",
    "solve_traditional", "split_index", "__version__",
]
