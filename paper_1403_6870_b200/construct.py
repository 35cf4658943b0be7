"""Modified-ziggurat table construction (CPU, offline).

Restates the reference's layer solver and the quantities derived from it, so
tables for another ``i_max`` (or a re-derivation of the shipped ones) come
from this package too.  Reference behaviour, with citations
(`zigfast/tables.py` unless noted):

* the two densities with their exact tail integrals and inverses
  (`densities.py:41-67`): exp(-x) (convex) and exp(-x^2/2) (not convex);
* layers: starting from f = 0, each layer solves x * (f(x) - f_prev) = M / i_max
  for its LARGER root (ternary search for the peak of the gap, then bisection
  to the last ulp on the right branch), until no root exists (`:130-225`);
* slot masses: the tail mass above the first layer and, per bounded box, the
  curve area above the box floor, from the exact complementary integral,
  normalised (`:228-244`);
* the exponential's rejection band epsilon_max: the largest gap between the
  box chord and the curve in box units over all boxes (bounded Brent search
  plus a 4097-point grid, `:272-311`);
* ``verify_tables``: every stored quantity re-derived, masses by adaptive
  quadrature (`:314-353`).

Bit-for-bit reproduction of the shipped fixtures is tested in
`tests/test_construct.py`.  The sampling kernels index layers by the word's
low byte, so only i_max = 256 tables can be uploaded; other sizes are for
analysis (as in the reference, whose kernels mask 8 bits too).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import CurvatureViolation, InvalidSpec, NonConvergence, QuadratureFailure
from .tables import EXPONENTIAL, HALF_NORMAL, ZigguratTables

_X0_FACTOR = 2.0  # x[0] is a finite placeholder, twice the tail start (never sampled)


@dataclass(frozen=True)
class DensitySpec:
    """A strictly decreasing density on [0, inf) with peak 1 at 0."""

    kind: str
    density: Callable[[float], float]
    cdf_complement: Callable[[float], float]   # exact integral over [x, inf)
    inverse: Callable[[float], float]          # inverse of density on (0, 1]
    total_mass: float
    convex: bool
    density_vec: Callable[[np.ndarray], np.ndarray]


def exponential() -> DensitySpec:
    return DensitySpec(EXPONENTIAL, lambda x: math.exp(-x), lambda x: math.exp(-x),
                       lambda f: -math.log(f), 1.0, True, lambda x: np.exp(-x))


def half_normal() -> DensitySpec:
    c = math.sqrt(math.pi / 2.0)
    return DensitySpec(HALF_NORMAL, lambda x: math.exp(-0.5 * x * x),
                       lambda x: c * math.erfc(x / math.sqrt(2.0)),
                       lambda f: math.sqrt(-2.0 * math.log(f)), c, False,
                       lambda x: np.exp(-0.5 * x * x))


def get(kind: str) -> DensitySpec:
    if kind == EXPONENTIAL:
        return exponential()
    if kind == HALF_NORMAL:
        return half_normal()
    raise ValueError(f"unknown density kind: {kind!r}")


def _bisect_to_ulp(fn, lo: float, hi: float) -> float:
    """Bisection until the bracket has no representable midpoint
    (`tables.py:107-127`)."""
    flo, fhi = fn(lo), fn(hi)
    if flo == 0.0:
        return lo
    if fhi == 0.0:
        return hi
    if (flo > 0.0) == (fhi > 0.0):
        raise NonConvergence(f"no sign change on [{lo!r}, {hi!r}]")
    while True:
        mid = 0.5 * (lo + hi)
        if mid <= lo or mid >= hi:
            return hi if abs(fhi) < abs(flo) else lo
        fmid = fn(mid)
        if fmid == 0.0:
            return mid
        if (fmid > 0.0) == (flo > 0.0):
            lo, flo = mid, fmid
        else:
            hi, fhi = mid, fmid


def _right_root(gap, hi: float) -> float | None:
    """Largest zero of the unimodal ``gap`` on (0, hi) (negative at both ends),
    or None when the peak stays <= 0: ternary search for the peak, then
    bisection on the right-hand branch."""
    a, b = 0.0, hi
    for _ in range(200):
        third = (b - a) / 3.0
        m1, m2 = a + third, b - third
        if gap(m1) < gap(m2):
            a = m1
        else:
            b = m2
        if b - a <= 1e-14 * max(1.0, b):
            break
    peak = 0.5 * (a + b)
    if gap(peak) <= 0.0:
        return None
    return _bisect_to_ulp(gap, peak, hi)


def _require_monotone(spec: DensitySpec) -> None:
    grid = np.linspace(0.0, spec.inverse(1e-12), 1024)
    vals = np.array([spec.density(x) for x in grid])
    if vals[0] != 1.0 or np.any(np.diff(vals) >= 0.0):
        raise InvalidSpec(f"density for {spec.kind!r} is not strictly decreasing from 1")


def overhang_areas(spec: DensitySpec, t: ZigguratTables) -> np.ndarray:
    """Unnormalised slot masses: [tail, box 1 .. box l_max] (closed form)."""
    comp = spec.cdf_complement
    xe, fe = t.x_ext, t.f_ext
    masses = np.empty(t.l_max + 1)
    masses[0] = comp(xe[1])
    for j in range(1, t.l_max + 1):
        masses[j] = (comp(xe[j + 1]) - comp(xe[j])) - (xe[j] - xe[j + 1]) * fe[j]
    if np.any(masses < -1e-15 * spec.total_mass):
        raise QuadratureFailure("negative overhang mass; tables inconsistent with density")
    return np.maximum(masses, 0.0)


def quadrature_overhang_areas(spec: DensitySpec, t: ZigguratTables,
                              tol: float = 1e-9) -> np.ndarray:
    """The same masses by adaptive quadrature (the verifier's independent check)."""
    from scipy import integrate
    xe, fe = t.x_ext, t.f_ext
    masses = np.empty(t.l_max + 1)
    val, err = integrate.quad(spec.density, xe[1], np.inf, epsabs=1e-13, epsrel=1e-13)
    if err > tol:
        raise QuadratureFailure(f"tail integral error {err:g} exceeds {tol:g}")
    masses[0] = val
    for j in range(1, t.l_max + 1):
        floor = fe[j]
        val, err = integrate.quad(lambda x: spec.density(x) - floor, xe[j + 1], xe[j],
                                  epsabs=1e-13, epsrel=1e-13)
        if err > tol:
            raise QuadratureFailure(f"box {j} integral error {err:g} exceeds {tol:g}")
        masses[j] = val
    return masses


def box_epsilon(pdf, xl: float, xr: float, fb: float, ft: float, pdf_vec=None) -> float:
    """Largest gap between the chord (xl, ft)-(xr, fb) and the curve, in unit
    box coordinates (the chord is 1 - t there); CurvatureViolation if the
    curve rises above the chord."""
    from scipy import optimize
    w, h = xr - xl, ft - fb

    def chord_gap(t: float) -> float:
        return (1.0 - t) - (pdf(xl + t * w) - fb) / h

    best = optimize.minimize_scalar(lambda t: -chord_gap(t), bounds=(0.0, 1.0),
                                    method="bounded", options={"xatol": 1e-13})
    eps = max(chord_gap(0.0), chord_gap(1.0), chord_gap(best.x))
    ts = np.linspace(0.0, 1.0, 4097)
    curve = pdf_vec(xl + ts * w) if pdf_vec is not None else np.array([pdf(xl + t * w) for t in ts])
    gaps = (1.0 - ts) - (curve - fb) / h
    if gaps.min() < -1e-9:
        raise CurvatureViolation("chord dips below the density inside an overhang box")
    return max(eps, float(gaps.max()))


def compute_epsilon(spec: DensitySpec, t: ZigguratTables) -> float:
    """epsilon_max: the widest rejection band over all bounded boxes."""
    worst = 0.0
    for j in range(1, t.l_max + 1):
        worst = max(worst, box_epsilon(spec.density, *t.box_bounds(j), pdf_vec=spec.density_vec))
    if not 0.0 < worst < 1.0:
        raise CurvatureViolation(f"epsilon out of range: {worst!r}")
    return float(worst)


def solve_layers(spec: DensitySpec, i_max: int = 256, tol: float = 1e-12) -> ZigguratTables:
    """The full layer stack and its derived quantities (tables.py:153-225)."""
    if i_max < 2 or i_max & (i_max - 1):
        raise ValueError(f"i_max must be a power of two >= 2, got {i_max}")
    if tol <= 0.0:
        raise ValueError("tol must be positive")
    _require_monotone(spec)
    slot = spec.total_mass / i_max
    xs, fs = [math.nan], [0.0]
    right_of_first = spec.inverse(min(slot, 0.5))
    while fs[-1] < 1.0:
        below = fs[-1]
        hi = spec.inverse(below) if below > 0.0 else max(right_of_first, 4.0 * abs(math.log(slot)))
        root = _right_root(lambda x, c=below: x * (spec.density(x) - c) - slot, hi)
        if root is None:
            break
        xs.append(root)
        fs.append(spec.density(root))
    l_max = len(xs) - 1
    if l_max < 1:
        raise NonConvergence("no layers fit under the density")
    xs[0] = _X0_FACTOR * xs[1]
    x, f = np.array(xs), np.array(fs)
    if np.max(np.abs(x[1:] * np.diff(f) - slot)) > tol * max(1.0, slot):
        raise NonConvergence("layer areas drifted beyond tolerance")
    shell = ZigguratTables(distribution=spec.kind, i_max=i_max, l_max=l_max,
                           total_mass=spec.total_mass, x=x, f=f, a=np.zeros(l_max + 1),
                           epsilon_max=0.0)
    masses = overhang_areas(spec, shell)
    eps = compute_epsilon(spec, shell) if spec.convex else 0.0
    return ZigguratTables(distribution=spec.kind, i_max=i_max, l_max=l_max,
                          total_mass=spec.total_mass, x=x, f=f, a=masses / masses.sum(),
                          epsilon_max=eps)


def build_tables(kind: str, i_max: int = 256, tol: float = 1e-12) -> ZigguratTables:
    """Solve the tables of a named density (tables.py:356-358)."""
    return solve_layers(get(kind), i_max, tol)


def verify_tables(t: ZigguratTables, tol: float = 1e-9) -> list[str]:
    """Re-derive every stored quantity; the list of violations (empty = ok)."""
    spec = get(t.distribution)
    slot = t.total_mass / t.i_max
    problems: list[str] = []
    if np.any(np.diff(t.x) >= 0.0):
        problems.append("x is not strictly decreasing")
    if np.any(np.diff(t.f) <= 0.0):
        problems.append("f is not strictly increasing")
    if t.f[-1] >= 1.0:
        problems.append("top layer height reaches the density peak")
    off = np.abs(t.x[1:] * np.diff(t.f) - slot) > tol * max(1.0, slot)
    if off.any():
        problems.append(f"{off.sum()} layer(s) deviate from slot area {slot:g}")
    for k in range(1, t.l_max + 1):
        if abs(spec.density(t.x[k]) - t.f[k]) > tol:
            problems.append(f"f[{k}] does not equal density(x[{k}])")
            break
    raw = quadrature_overhang_areas(spec, t)
    total = t.l_max * slot + raw.sum()
    if abs(total - t.total_mass) > 1e-9 * t.total_mass:
        problems.append(f"mass not conserved: {total!r} vs {t.total_mass!r}")
    if np.max(np.abs(raw / raw.sum() - t.a)) > 1e-9:
        problems.append("stored slot masses disagree with quadrature")
    if spec.convex:
        eps = compute_epsilon(spec, t)
        if abs(eps - t.epsilon_max) > 1e-9:
            problems.append(f"epsilon_max mismatch: {eps!r} vs {t.epsilon_max!r}")
    return problems
