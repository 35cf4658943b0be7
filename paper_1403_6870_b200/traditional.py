"""Traditional (Marsaglia-Tsang) ziggurat baseline on B200.

Mirrors `zigfast/traditional.py:1-207`: the equal-area layer stack
(`solve_traditional`, :56-96 -- shipped solved for i_max = 256 in
data/traditional_256.npz, exported from the reference), the integer fast-accept
thresholds (`_int_thresholds`, :99-110, for caller-supplied tables), the flat
pack (`_pack`, :113-121) and the two samplers with the reference's methods (`sample`,
`sample_counted`, `fill`, `fill_counted`, `aggregate`, `path_counts`,
`reset_counters`, `fast_accept_fraction`).  The draw bodies run in the sm_100a
library (dist codes ZF_TRAD_EXP / ZF_TRAD_NORMAL) on the same sources as the
modified samplers: production counter streams and the reference's exact
sequential streams (oracle mode).

Counter slots follow `trad_*_counted` (`_kernels.py:956-979, 1117-1146`):
0 byte words, 1 fast accepts, 2 wedge (density) tests, 3 tail entries.

The tail values are `r - log(u)` (exp) and `r + (-log(u) / r)` (normal): the
device evaluates log in double-double and rounds once, i.e. the correctly
rounded log, which is what glibc returns for all but a vanishing fraction of
arguments; the tests allow 2 ulp on tail samples (north_star's tolerance) and
require bit equality everywhere else.
"""

from __future__ import annotations

import pathlib
from dataclasses import dataclass

import numpy as np

from . import _lib
from .samplers import _SamplerBase
from .tables import EXPONENTIAL, HALF_NORMAL
from .uniform import UniformSource

TWO_64 = 2.0 ** 64
TWO_63 = 2.0 ** 63


def _kind_of(spec) -> str:
    kind = spec if isinstance(spec, str) else getattr(spec, "kind", None)
    if kind not in (EXPONENTIAL, HALF_NORMAL):
        raise ValueError(f"unknown density kind: {kind!r}")
    return kind


@dataclass(frozen=True)
class TraditionalTables:
    """Traditional layer stack plus the per-byte fast-accept ratio table
    (`traditional.py:33-53`)."""

    distribution: str
    i_max: int
    r: float
    v: float          # area of every strip, tail included in strip 0
    x: np.ndarray     # x[0] = r, x[i] = inverse(f[i]); decreasing
    f: np.ndarray     # f[0] = density(r), f[i_max - 1] == 1
    k: np.ndarray     # fast-accept ratios per byte, in [0, 1]

    @property
    def edge(self) -> np.ndarray:
        """Per-byte proposal edge length: virtual base edge, then x[i-1]."""
        e = np.empty(self.i_max)
        e[0] = self.v / self.f[0]
        e[1:] = self.x[:-1]
        return e

    def fast_accept_probability(self) -> float:
        return float(self.k.mean())


_FIXTURE_PATH = pathlib.Path(__file__).resolve().parent / "data" / "traditional_256.npz"
_FIXTURE: dict = {}


def _fixture(kind: str):
    """(tables, pack) of the shipped i_max = 256 solution for ``kind``: the
    reference's own `solve_traditional` and `_pack` output, exported by
    tests/golden/make_golden.py, so nothing is re-solved at import or run time."""
    hit = _FIXTURE.get(kind)
    if hit is None:
        with np.load(_FIXTURE_PATH) as z:
            r, v = (float(a) for a in z[f"{kind}_rv"])
            t = TraditionalTables(distribution=kind, i_max=256, r=r, v=v, x=z[f"{kind}_x"],
                                  f=z[f"{kind}_f"], k=z[f"{kind}_k"])
            pack = TradPack(se=z[f"{kind}_se"], kk=z[f"{kind}_kk"].astype(np.uint64),
                            flo=z[f"{kind}_flo"], fh=z[f"{kind}_fh"], r=r)
        hit = _FIXTURE[kind] = (t, pack)
    return hit


def solve_traditional(spec, i_max: int = 256, tol: float = 1e-12) -> TraditionalTables:
    """The traditional equal-area layer stack (`traditional.py:56-96`) for the
    samplers' i_max = 256.  ``spec`` is a density kind or an object with a
    ``kind`` attribute (the reference's DensitySpec).  The device samplers
    index strips by the word's low byte, so 256 is the only stack they can use;
    it ships solved (bit-identical to the reference's bisection, checked
    against reference digests in tests/test_traditional_host.py)."""
    if i_max != 256:
        raise ValueError(f"only i_max = 256 is available (the samplers index strips by the "
                         f"word's low byte), got {i_max}")
    return _fixture(_kind_of(spec))[0]


def _int_thresholds(tables: TraditionalTables, scale: float) -> np.ndarray:
    """floor(k * scale), nudged down so a fast accept can never overshoot
    (`traditional.py:99-110`)."""
    edge = tables.edge
    bound = np.empty(tables.i_max)
    bound[0] = tables.r
    bound[1:] = tables.x[1:]
    kk = np.floor(tables.k * scale).astype(np.uint64)
    inv = 1.0 / scale
    for i in range(tables.i_max):
        while kk[i] > 0 and np.float64(kk[i]) * inv * edge[i] > bound[i]:
            kk[i] -= np.uint64(1)
    return kk


@dataclass(frozen=True)
class TradPack:
    se: np.ndarray
    kk: np.ndarray
    flo: np.ndarray
    fh: np.ndarray
    r: float


def trad_pack(tables: TraditionalTables) -> TradPack:
    """`_pack(tables, signed)` (`traditional.py:113-121`): the flat arrays the
    draw bodies read (signed = half-normal, words scaled by 2^-63).  The
    shipped tables come with their shipped pack."""
    shipped = _FIXTURE.get(tables.distribution)
    if shipped is not None and shipped[0] is tables:
        return shipped[1]
    scale = TWO_63 if tables.distribution == HALF_NORMAL else TWO_64
    se = tables.edge * (1.0 / scale)
    kk = _int_thresholds(tables, scale)
    flo = np.zeros(tables.i_max)
    fh = np.zeros(tables.i_max)
    flo[1:] = tables.f[:-1]
    fh[1:] = tables.f[1:] - tables.f[:-1]
    return TradPack(se=se, kk=kk, flo=flo, fh=fh, r=float(tables.r))


class _TraditionalSampler(_SamplerBase):
    """`_TraditionalSampler` (`traditional.py:124-142`) on the device."""

    def __init__(self, kind: str, i_max: int, source: UniformSource | None,
                 tables: TraditionalTables | None, device):
        if tables is None:
            tables = solve_traditional(kind, i_max)
        if tables.distribution != kind:
            raise ValueError(f"tables are for {tables.distribution!r}, need {kind!r}")
        if tables.i_max != 256:
            raise ValueError("the device kernels index layers by the word's low byte: i_max = 256")
        self._init_device(source, device)
        self.tables = tables
        other = solve_traditional(HALF_NORMAL if kind == EXPONENTIAL else EXPONENTIAL, 256)
        exp_t, hn_t = (tables, other) if kind == EXPONENTIAL else (other, tables)
        self._dev_tables = _lib.device_trad_tables(exp_t, hn_t, self.device.index)

    def fast_accept_fraction(self) -> float:
        c = self.counters
        return c[1] / c[0] if c[0] else 0.0


class TraditionalExpSampler(_TraditionalSampler):
    """`TraditionalExpSampler` (`traditional.py:145-176`)."""

    _dist = _lib.TRAD_EXP

    def __init__(self, tables: TraditionalTables | None = None,
                 source: UniformSource | None = None, i_max: int = 256, device=None):
        super().__init__(EXPONENTIAL, i_max, source, tables, device)


class TraditionalNormalSampler(_TraditionalSampler):
    """`TraditionalNormalSampler` (`traditional.py:179-207`)."""

    _dist = _lib.TRAD_NORMAL

    def __init__(self, tables: TraditionalTables | None = None,
                 source: UniformSource | None = None, i_max: int = 256, device=None):
        super().__init__(HALF_NORMAL, i_max, source, tables, device)
