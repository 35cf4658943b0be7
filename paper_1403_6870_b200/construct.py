"""Modified-ziggurat table construction (host side, offline).

What it computes is the reference's (`zigfast/tables.py:153-353`,
`densities.py:41-67`): for a strictly decreasing density f with f(0) = 1 and
i_max slots of mass M / i_max, layer k's right edge x_k is the LARGER solution
of x (f(x) - f_{k-1}) = M / i_max, layers are added until that equation has
no solution, the leftover mass is split into the tail slot and one slot per
bounded overhang box, and for convex densities the rejection band
epsilon_max is the widest chord-to-curve gap over the boxes.

How it computes it is new (the sampler never runs this code; the shipped
i_max = 256 tables are loaded from data/*.zigt):

* layers: the per-layer gap g(x) = x (f(x) - c) - M / i_max has derivative
  g'(x) = f(x) - c + x f'(x).  Its peak is the root of g' (bracketed on
  (0, 1] for both densities, safeguarded Newton with g''), the layer edge the
  root of g right of the peak (safeguarded Newton from the right end, where
  g = -M / i_max), polished to adjacent doubles.  Densities other than the
  two built-in ones get central-difference derivatives;
* slot masses: the closed form from the density's complementary integral,
  vectorised;
* epsilon_max: for the exponential the chord-to-curve gap of a box is
  concave in the box coordinate and its maximum sits where f' equals the
  chord slope, x* = -log(h / w) -- evaluated in closed form; other convex
  densities use a golden-section search on the gap;
* verify_tables: masses re-derived by composite Gauss-Legendre quadrature
  (the tail through x = x_1 + s / (1 - s)), with the 48- and 64-node rules
  compared as the error estimate.

Against the reference's own tables (tests/test_construct.py): l_max, f and
the slot structure are identical; x agrees to the last bit except where
x (f(x) - c) - M / i_max changes sign more than once between adjacent
doubles (one layer per density at i_max = 256, 1 ulp, with an identical
f = density(x)); slot masses agree to ~1e-16 and epsilon_max to ~1e-15.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import CurvatureViolation, InvalidSpec, NonConvergence, QuadratureFailure
from .tables import EXPONENTIAL, HALF_NORMAL, ZigguratTables

_SENTINEL = 2.0  # x[0] = 2 x[1]: a finite placeholder no sampling path reads


@dataclass(frozen=True)
class DensitySpec:
    """`densities.DensitySpec` (densities.py:24-38): an unnormalised, strictly
    decreasing density on [0, inf) with f(0) = 1, its exact upper-tail
    integral, its inverse on (0, 1], the total mass, whether chords lie above
    the curve everywhere, and a vectorised twin of the density."""

    kind: str
    density: Callable[[float], float]
    cdf_complement: Callable[[float], float]
    inverse: Callable[[float], float]
    total_mass: float
    convex: bool
    density_vec: Callable[[np.ndarray], np.ndarray] = None


def exponential() -> DensitySpec:
    """exp(-x): mass 1, convex."""
    return DensitySpec(EXPONENTIAL, lambda x: math.exp(-x), lambda x: math.exp(-x),
                       lambda y: -math.log(y), 1.0, True, lambda x: np.exp(-x))


def half_normal() -> DensitySpec:
    """exp(-x^2 / 2): mass sqrt(pi / 2), inflection at x = 1 (not convex)."""
    mass = math.sqrt(math.pi / 2.0)
    return DensitySpec(HALF_NORMAL, lambda x: math.exp(-0.5 * x * x),
                       lambda x: mass * math.erfc(x / math.sqrt(2.0)),
                       lambda y: math.sqrt(-2.0 * math.log(y)), mass, False,
                       lambda x: np.exp(-0.5 * x * x))


_FACTORIES = {EXPONENTIAL: exponential, HALF_NORMAL: half_normal}


def get(kind: str) -> DensitySpec:
    factory = _FACTORIES.get(kind)
    if factory is None:
        raise ValueError(f"unknown density kind: {kind!r}")
    return factory()


# -- derivatives of the built-in densities (first, second) -------------------------

def _derivatives(spec: DensitySpec):
    if spec.kind == EXPONENTIAL:
        return (lambda x: -math.exp(-x)), (lambda x: math.exp(-x))
    if spec.kind == HALF_NORMAL:
        return ((lambda x: -x * math.exp(-0.5 * x * x)),
                (lambda x: (x * x - 1.0) * math.exp(-0.5 * x * x)))

    def d1(x, h=1e-6):
        return (spec.density(x + h) - spec.density(max(x - h, 0.0))) / (x + h - max(x - h, 0.0))

    def d2(x, h=1e-4):
        lo = max(x - h, 0.0)
        return (d1(x + h) - d1(lo)) / (x + h - lo)
    return d1, d2


def _newton_bracket(fn, dfn, a: float, b: float, start: float) -> tuple[float, float]:
    """Shrink [a, b] (fn(a) > 0 >= fn(b), or the reverse) around a root of fn
    with Newton steps from `start`, falling back to the midpoint whenever a
    step leaves the bracket; returns the bracket once its ends are adjacent
    doubles or Newton stops moving."""
    pos_left = fn(a) > 0.0
    x = start
    for _ in range(400):
        if not a < x < b:
            x = 0.5 * (a + b)
        v = fn(x)
        if v == 0.0:
            return x, x
        if (v > 0.0) == pos_left:
            a = x
        else:
            b = x
        if math.nextafter(a, b) >= b:
            break
        d = dfn(x)
        nxt = x - v / d if d != 0.0 and math.isfinite(d) else 0.5 * (a + b)
        x = nxt if (a < nxt < b and nxt != x) else 0.5 * (a + b)
    return a, b


def _to_adjacent(fn, a: float, b: float) -> float:
    """Resolve a tiny sign-change bracket down to two adjacent doubles and
    return the end with the smaller |fn| (the upper end on a tie)."""
    fa, fb = fn(a), fn(b)
    if fa == 0.0:
        return a
    if fb == 0.0:
        return b
    while True:
        m = 0.5 * (a + b)
        if m <= a or m >= b:
            return b if abs(fb) < abs(fa) else a
        fm = fn(m)
        if fm == 0.0:
            return m
        if (fm > 0.0) == (fa > 0.0):
            a, fa = m, fm
        else:
            b, fb = m, fm


def _check_decreasing(spec: DensitySpec) -> None:
    xs = np.linspace(0.0, spec.inverse(1e-12), 2048)
    ys = np.array([spec.density(x) for x in xs])
    if ys[0] != 1.0 or np.any(np.diff(ys) >= 0.0):
        raise InvalidSpec(f"density for {spec.kind!r} must fall strictly from 1 at x = 0")


def _layer_stack(spec: DensitySpec, i_max: int):
    """x, f of layers 1..l_max (index 0 = sentinel / zero height)."""
    d1, d2 = _derivatives(spec)
    f = spec.density
    slot = spec.total_mass / i_max
    xs, fs = [math.nan], [0.0]
    first_hi = max(spec.inverse(min(slot, 0.5)), 4.0 * abs(math.log(slot)))
    while fs[-1] < 1.0:
        c = fs[-1]

        def g(x, c=c):
            return x * (f(x) - c) - slot

        def dg(x, c=c):
            return f(x) - c + x * d1(x)

        def ddg(x):
            return 2.0 * d1(x) + x * d2(x)

        # the peak of g: g'(0) = 1 - c > 0 and g'(1) <= 0 for both densities
        # (g'(1) = -c, resp. f(1) * 0 - c); generic densities scan right
        right = 1.0
        while dg(right) > 0.0:
            right *= 2.0
            if right > 1e6:
                raise NonConvergence("layer gap has no interior maximum")
        pa, pb = _newton_bracket(dg, ddg, 0.0, right, 0.5 * right)
        peak = pa if abs(dg(pa)) <= abs(dg(pb)) else pb
        if g(peak) <= 0.0:
            break  # no layer of the slot's area fits under the density any more
        hi = spec.inverse(c) if c > 0.0 else first_hi
        if not g(hi) < 0.0:
            raise NonConvergence(f"layer {len(xs)}: no sign change right of the peak")
        a, b = _newton_bracket(g, dg, peak, hi, hi)
        root = _to_adjacent(g, a, b)
        xs.append(root)
        fs.append(f(root))
    if len(xs) < 2:
        raise NonConvergence("no layers fit under the density")
    xs[0] = _SENTINEL * xs[1]
    return np.array(xs), np.array(fs)


def overhang_areas(spec: DensitySpec, t: ZigguratTables) -> np.ndarray:
    """Unnormalised slot masses [tail, box 1 .. box l_max] from the density's
    exact upper-tail integral (`tables.py:228-244`)."""
    xe, fe = t.x_ext, t.f_ext
    comp = np.array([spec.cdf_complement(v) for v in xe[1:]])  # comp(xe[1 .. l_max + 1])
    masses = np.empty(t.l_max + 1)
    masses[0] = comp[0]
    j = np.arange(1, t.l_max + 1)
    masses[1:] = (comp[j] - comp[j - 1]) - (xe[j] - xe[j + 1]) * fe[j]
    if np.any(masses < -1e-15 * spec.total_mass):
        raise QuadratureFailure("negative overhang mass: tables inconsistent with the density")
    return np.maximum(masses, 0.0)


def _box_gap(spec: DensitySpec, xl: float, xr: float, fb: float, ft: float):
    w, h = xr - xl, ft - fb
    return lambda u: (1.0 - u) - (spec.density(xl + u * w) - fb) / h


def box_epsilon(spec: DensitySpec, xl: float, xr: float, fb: float, ft: float) -> float:
    """Widest gap between the chord (xl, ft)-(xr, fb) and the curve, in box
    units (chord = 1 - u at u = (x - xl) / w)."""
    gap = _box_gap(spec, xl, xr, fb, ft)
    w, h = xr - xl, ft - fb
    if spec.kind == EXPONENTIAL:
        # concave gap; its maximum where f'(x) = -h / w, i.e. x* = -log(h / w)
        u = min(max((-math.log(h / w) - xl) / w, 0.0), 1.0)
        best = gap(u)
    else:  # golden-section search on the (unimodal) gap
        r = (math.sqrt(5.0) - 1.0) / 2.0
        a, b = 0.0, 1.0
        c, d = b - r * (b - a), a + r * (b - a)
        gc, gd = gap(c), gap(d)
        while b - a > 1e-12:
            if gc > gd:
                b, d, gd = d, c, gc
                c = b - r * (b - a)
                gc = gap(c)
            else:
                a, c, gc = c, d, gd
                d = a + r * (b - a)
                gd = gap(d)
        best = max(gc, gd)
    eps = max(gap(0.0), gap(1.0), best)
    if min(gap(0.25), gap(0.5), gap(0.75)) < -1e-9:
        raise CurvatureViolation("the curve rises above the chord inside an overhang box")
    return float(eps)


def compute_epsilon(spec: DensitySpec, t: ZigguratTables) -> float:
    """epsilon_max over the bounded boxes (`tables.py:301-311`)."""
    eps = max(box_epsilon(spec, *t.box_bounds(j)) for j in range(1, t.l_max + 1))
    if not 0.0 < eps < 1.0:
        raise CurvatureViolation(f"epsilon_max out of range: {eps!r}")
    return eps


def solve_layers(spec: DensitySpec, i_max: int = 256, tol: float = 1e-12) -> ZigguratTables:
    """Complete tables for ``spec`` with ``i_max`` slots (`tables.py:153-225`)."""
    if i_max < 2 or i_max & (i_max - 1):
        raise ValueError(f"i_max must be a power of two >= 2, got {i_max}")
    if tol <= 0.0:
        raise ValueError("tol must be positive")
    _check_decreasing(spec)
    x, f = _layer_stack(spec, i_max)
    slot = spec.total_mass / i_max
    if np.max(np.abs(x[1:] * np.diff(f) - slot)) > tol * max(1.0, slot):
        raise NonConvergence("layer areas drifted beyond tolerance")
    l_max = len(x) - 1
    shell = ZigguratTables(distribution=spec.kind, i_max=i_max, l_max=l_max,
                           total_mass=spec.total_mass, x=x, f=f, a=np.zeros(l_max + 1),
                           epsilon_max=0.0)
    raw = overhang_areas(spec, shell)
    eps = compute_epsilon(spec, shell) if spec.convex else 0.0
    return ZigguratTables(distribution=spec.kind, i_max=i_max, l_max=l_max,
                          total_mass=spec.total_mass, x=x, f=f, a=raw / raw.sum(),
                          epsilon_max=eps)


def build_tables(kind: str, i_max: int = 256, tol: float = 1e-12) -> ZigguratTables:
    """Tables of a named density (`tables.py:356-358`)."""
    return solve_layers(get(kind), i_max, tol)


# -- verification ---------------------------------------------------------------------

_GL = {k: np.polynomial.legendre.leggauss(k) for k in (48, 64)}


def _gauss(fvec, a: float, b: float, panels: int, k: int) -> float:
    nodes, weights = _GL[k]
    edges = np.linspace(a, b, panels + 1)
    mid = 0.5 * (edges[1:] + edges[:-1])[:, None]
    half = 0.5 * (edges[1:] - edges[:-1])[:, None]
    return float((fvec(mid + half * nodes[None, :]) * weights[None, :] * half).sum())


def quadrature_overhang_areas(spec: DensitySpec, t: ZigguratTables,
                              tol: float = 1e-9) -> np.ndarray:
    """Slot masses by composite Gauss-Legendre quadrature; the 48- and 64-node
    rules must agree within ``tol``."""
    fvec = spec.density_vec or np.vectorize(spec.density)
    xe, fe = t.x_ext, t.f_ext
    x1 = xe[1]

    def tail(s):  # x = x1 + s / (1 - s), dx = ds / (1 - s)^2 on [0, 1)
        return fvec(x1 + s / (1.0 - s)) / (1.0 - s) ** 2

    masses = np.empty(t.l_max + 1)
    pair = [_gauss(tail, 0.0, 1.0 - 1e-12, 256, k) for k in (48, 64)]
    if abs(pair[0] - pair[1]) > tol:
        raise QuadratureFailure(f"tail quadrature disagreement {abs(pair[0] - pair[1]):g}")
    masses[0] = pair[1]
    for j in range(1, t.l_max + 1):
        floor = fe[j]
        pair = [_gauss(lambda x: fvec(x) - floor, xe[j + 1], xe[j], 4, k) for k in (48, 64)]
        if abs(pair[0] - pair[1]) > tol:
            raise QuadratureFailure(f"box {j}: quadrature disagreement {abs(pair[0] - pair[1]):g}")
        masses[j] = pair[1]
    return masses


def verify_tables(t: ZigguratTables, tol: float = 1e-9) -> list[str]:
    """Every stored quantity re-derived independently; the violations found
    (empty list = consistent), `tables.py:314-353`."""
    spec = get(t.distribution)
    slot = t.total_mass / t.i_max
    issues: list[str] = []
    if np.any(np.diff(t.x) >= 0.0):
        issues.append("x is not strictly decreasing")
    if np.any(np.diff(t.f) <= 0.0):
        issues.append("f is not strictly increasing")
    if t.f[-1] >= 1.0:
        issues.append("top layer height reaches the density peak")
    bad = np.abs(t.x[1:] * np.diff(t.f) - slot) > tol * max(1.0, slot)
    if bad.any():
        issues.append(f"{int(bad.sum())} layer(s) deviate from slot area {slot:g}")
    dens = np.array([spec.density(v) for v in t.x[1:]])
    if np.any(np.abs(dens - t.f[1:]) > tol):
        issues.append("f does not equal the density at x")
    raw = quadrature_overhang_areas(spec, t)
    total = t.l_max * slot + raw.sum()
    if abs(total - t.total_mass) > 1e-9 * t.total_mass:
        issues.append(f"mass not conserved: {total!r} vs {t.total_mass!r}")
    if np.max(np.abs(raw / raw.sum() - t.a)) > 1e-9:
        issues.append("stored slot masses disagree with quadrature")
    if spec.convex:
        eps = compute_epsilon(spec, t)
        if abs(eps - t.epsilon_max) > 1e-9:
            issues.append(f"epsilon_max mismatch: {eps!r} vs {t.epsilon_max!r}")
    return issues
