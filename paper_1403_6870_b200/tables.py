"""Ziggurat table data, its two on-disk formats, and the Walker/Vose alias.

Only the *data* half of the reference's table layer lives here: the tables
are consumed exactly as the reference ships them (i_max = 256), the layer
solver (`zigfast/tables.py:107-353`) stays offline and out of scope.

Reference behaviour mirrored, with citations:

* slot convention and the cap extension `x_ext/f_ext`   `tables.py:10-18,69-75`
* `scaled_x = x * 2**-64`                                 `tables.py:60-65`
* JSON with C99 hex floats + CRC32 over the canonical dump `tableio.py:43-94`
* binary `ZIGT` container                                 `tableio.py:97-143`
* Vose alias build with LIFO work lists                    `alias.py:32-63`
* per-slot overhang box arrays                            `_packs.py:15-28`

The package ships the two reference tables re-serialised in the binary
`ZIGT` form (`data/*.zigt`, produced by `tools/export_tables.py`); both
formats load through :func:`load` / :func:`from_json_bytes`.
"""

from __future__ import annotations

import json
import math
import struct
import zlib
from dataclasses import dataclass, field
from importlib import resources

import numpy as np

from .errors import EmptyWeights, FormatError

EXPONENTIAL = "exponential"
HALF_NORMAL = "halfnormal"

TWO_NEG_64 = 2.0 ** -64
TWO_NEG_63 = 2.0 ** -63

SCHEMA_VERSION = 1
_MAGIC = b"ZIGT"
_DIST_CODE = {EXPONENTIAL: 0, HALF_NORMAL: 1}
_CODE_DIST = {code: name for name, code in _DIST_CODE.items()}
_HEADER = struct.Struct("<4sBBII")
_SCALARS = struct.Struct("<2d")


@dataclass(frozen=True)
class ZigguratTables:
    """Layer geometry for one density (`tables.py:39-104`).

    ``x``/``f`` hold ``l_max + 1`` entries (``x[0]`` is a finite sentinel
    that no sampling path reads), ``a`` the ``l_max + 1`` slot masses.
    """

    distribution: str
    i_max: int
    l_max: int
    total_mass: float
    x: np.ndarray
    f: np.ndarray
    a: np.ndarray
    epsilon_max: float
    scaled_x: np.ndarray = field(init=False, repr=False)
    scaled_f: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        for name in ("x", "f", "a"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        object.__setattr__(self, "scaled_x", self.x * TWO_NEG_64)
        object.__setattr__(self, "scaled_f", self.f * TWO_NEG_64)

    @property
    def x_ext(self) -> np.ndarray:
        """X with the cap's virtual right edge (0.0) appended."""
        return np.concatenate([self.x, [0.0]])

    @property
    def f_ext(self) -> np.ndarray:
        """F with the cap's virtual top (density(0) = 1.0) appended."""
        return np.concatenate([self.f, [1.0]])

    def box_bounds(self, j: int):
        """``(x_left, x_right, f_bottom, f_top)`` of bounded slot ``j``."""
        if not 1 <= j <= self.l_max:
            raise IndexError(f"bounded box index out of range: {j}")
        xe, fe = self.x_ext, self.f_ext
        return xe[j + 1], xe[j], fe[j], fe[j + 1]

    def __eq__(self, other) -> bool:
        if not isinstance(other, ZigguratTables):
            return NotImplemented
        same_scalars = (self.distribution, self.i_max, self.l_max, self.total_mass,
                        self.epsilon_max) == (other.distribution, other.i_max, other.l_max,
                                              other.total_mass, other.epsilon_max)
        return same_scalars and all(
            np.array_equal(getattr(self, k), getattr(other, k)) for k in ("x", "f", "a"))

    __hash__ = None


# ---------------------------------------------------------------------------
# serialisation
# ---------------------------------------------------------------------------

def _hexfloat(v: float) -> str:
    return "inf" if math.isinf(v) else float(v).hex()


def _parse_hex(text) -> float:
    try:
        return float.fromhex(text)
    except (TypeError, ValueError) as exc:
        raise FormatError(f"bad float field: {text!r}") from exc


def _canonical(t: ZigguratTables) -> dict:
    return {
        "schema_version": SCHEMA_VERSION,
        "distribution": t.distribution,
        "i_max": t.i_max,
        "L_max": t.l_max,
        "total_mass": _hexfloat(t.total_mass),
        "X": [_hexfloat(v) for v in t.x],
        "F": [_hexfloat(v) for v in t.f],
        "A": [_hexfloat(v) for v in t.a],
        "epsilon_max": _hexfloat(t.epsilon_max),
    }


def _crc_of(doc: dict) -> str:
    # the checksum covers the sorted, whitespace-free dump (tableio.py:57-59)
    return "%08x" % zlib.crc32(json.dumps(doc, sort_keys=True, separators=(",", ":")).encode())


def to_json_bytes(t: ZigguratTables) -> bytes:
    doc = _canonical(t)
    doc["checksum"] = _crc_of(doc)
    return (json.dumps(doc, indent=1) + "\n").encode()


def from_json_bytes(data: bytes) -> ZigguratTables:
    try:
        doc = json.loads(data)
    except json.JSONDecodeError as exc:
        raise FormatError("not valid JSON") from exc
    if not isinstance(doc, dict):
        raise FormatError("table file must be a JSON object")
    if doc.get("schema_version") != SCHEMA_VERSION:
        raise FormatError(f"unsupported schema_version: {doc.get('schema_version')!r}")
    stored = doc.pop("checksum", None)
    if stored is None or _crc_of(doc) != stored:
        raise FormatError("checksum mismatch")
    if doc.get("distribution") not in _DIST_CODE:
        raise FormatError(f"unknown distribution: {doc.get('distribution')!r}")
    try:
        return ZigguratTables(
            distribution=doc["distribution"], i_max=int(doc["i_max"]), l_max=int(doc["L_max"]),
            total_mass=_parse_hex(doc["total_mass"]),
            x=np.array([_parse_hex(v) for v in doc["X"]]),
            f=np.array([_parse_hex(v) for v in doc["F"]]),
            a=np.array([_parse_hex(v) for v in doc["A"]]),
            epsilon_max=_parse_hex(doc["epsilon_max"]))
    except KeyError as exc:
        raise FormatError(f"missing field: {exc}") from exc


def to_binary(t: ZigguratTables) -> bytes:
    n = t.l_max + 1
    body = _HEADER.pack(_MAGIC, SCHEMA_VERSION, _DIST_CODE[t.distribution], t.i_max, t.l_max)
    body += _SCALARS.pack(t.total_mass, t.epsilon_max)
    body += b"".join(np.asarray(arr, dtype="<f8").tobytes() for arr in (t.x, t.f, t.a))
    assert all(len(arr) == n for arr in (t.x, t.f, t.a))
    return body + struct.pack("<I", zlib.crc32(body))


def from_binary(data: bytes) -> ZigguratTables:
    if len(data) < _HEADER.size + 4 or data[:4] != _MAGIC:
        raise FormatError("missing ZIGT magic")
    body = data[:-4]
    (crc,) = struct.unpack("<I", data[-4:])
    if zlib.crc32(body) != crc:
        raise FormatError("checksum mismatch")
    _, version, code, i_max, l_max = _HEADER.unpack_from(body, 0)
    if version != SCHEMA_VERSION:
        raise FormatError(f"unsupported version byte: {version}")
    if code not in _CODE_DIST:
        raise FormatError(f"unknown distribution code: {code}")
    n = l_max + 1
    off = _HEADER.size + _SCALARS.size
    if len(body) != off + 3 * 8 * n:
        raise FormatError("truncated or oversized table body")
    total_mass, eps = _SCALARS.unpack_from(body, _HEADER.size)
    arrays = [np.frombuffer(body, dtype="<f8", count=n, offset=off + 8 * n * k).astype(np.float64)
              for k in range(3)]
    return ZigguratTables(distribution=_CODE_DIST[code], i_max=i_max, l_max=l_max,
                          total_mass=total_mass, x=arrays[0], f=arrays[1], a=arrays[2],
                          epsilon_max=eps)


def save(t: ZigguratTables, path, fmt: str = "json") -> None:
    with open(path, "wb") as fh:
        fh.write(to_json_bytes(t) if fmt == "json" else to_binary(t))


def load(path) -> ZigguratTables:
    with open(path, "rb") as fh:
        data = fh.read()
    return from_binary(data) if data[:4] == _MAGIC else from_json_bytes(data)


_DEFAULTS: dict[str, ZigguratTables] = {}


def default_tables(kind: str) -> ZigguratTables:
    """The shipped i_max = 256 tables for ``kind`` (`tables.py:359-372`)."""
    if kind not in _DIST_CODE:
        raise ValueError(f"unknown density kind: {kind!r}")
    if kind not in _DEFAULTS:
        blob = resources.files(__package__).joinpath("data", f"{kind}_256.zigt").read_bytes()
        _DEFAULTS[kind] = from_binary(blob)
    return _DEFAULTS[kind]


# ---------------------------------------------------------------------------
# alias table
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class AliasTable:
    """Walker alias arrays: one index uniform plus one acceptance uniform."""

    size: int
    prob: np.ndarray
    alias: np.ndarray

    def sample(self, u_index: float, u_prob: float) -> int:
        k = min(int(u_index * self.size), self.size - 1)
        return k if u_prob < self.prob[k] else int(self.alias[k])

    def exact_probabilities(self) -> np.ndarray:
        out = self.prob.copy()
        np.add.at(out, self.alias, 1.0 - self.prob)
        return out / self.size


def build_alias(weights) -> AliasTable:
    """Vose's worklist construction, bit-compatible with `alias.py:32-63`.

    The device consumes these arrays verbatim, so the floating-point update
    ``(big + small) - 1`` and the last-in-first-out order of both work lists
    must match the reference exactly: a different pairing gives a different
    (equally valid) table and therefore a different draw stream.
    """
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or w.size == 0:
        raise ValueError("weights must be a nonempty 1-D array")
    if not np.all(np.isfinite(w)) or np.any(w < 0.0):
        raise ValueError("weights must be finite and nonnegative")
    total = w.sum()
    if total <= 0.0:
        raise EmptyWeights("all weights are zero")
    n = w.size
    level = w * (n / total)
    prob = np.ones(n)
    alias = np.arange(n, dtype=np.int64)
    below = [k for k in range(n) if level[k] < 1.0]
    above = [k for k in range(n) if level[k] >= 1.0]
    while below and above:
        lo, hi = below.pop(), above.pop()
        prob[lo] = level[lo]
        alias[lo] = hi
        level[hi] = (level[hi] + level[lo]) - 1.0
        (below if level[hi] < 1.0 else above).append(hi)
    for k in below + above:          # numerically-1 leftovers
        prob[k] = 1.0
    return AliasTable(size=n, prob=prob, alias=alias)


# ---------------------------------------------------------------------------
# flat packs handed to the device (layout of `_packs.py:15-60`)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SamplerPack:
    """Everything one distribution's draw body reads, as float64/int64 arrays.

    ``scale`` is the fast-path multiplier table: ``X * 2**-64`` for the
    exponential's unsigned word, ``X * 2**-63`` for the normal's signed word.
    Box arrays have ``l_max + 1`` entries with slot 0 (the tail) unused.
    """

    kind: str
    l_max: int
    scale: np.ndarray
    xlo: np.ndarray
    xw: np.ndarray
    flo: np.ndarray
    fh: np.ndarray
    eps: float
    prob: np.ndarray
    alias: np.ndarray
    tail_x: float


def overhang_arrays(t: ZigguratTables):
    """Slot j box = ``[x_ext[j+1], x_ext[j]] x [f_ext[j], f_ext[j+1]]``."""
    xe, fe = t.x_ext, t.f_ext
    slots = np.arange(1, t.l_max + 1)
    xlo, xw, flo, fh = (np.zeros(t.l_max + 1) for _ in range(4))
    xlo[slots] = xe[slots + 1]
    xw[slots] = xe[slots] - xe[slots + 1]
    flo[slots] = fe[slots]
    fh[slots] = fe[slots + 1] - fe[slots]
    return xlo, xw, flo, fh


def make_pack(t: ZigguratTables, alias: AliasTable | None = None) -> SamplerPack:
    alias = alias if alias is not None else build_alias(t.a)
    xlo, xw, flo, fh = overhang_arrays(t)
    if t.distribution == EXPONENTIAL:
        scale, eps = t.scaled_x, float(t.epsilon_max)
    else:
        # normal pack carries no band: plain rejection in every box (_packs.py:47-60)
        scale, eps = t.x * TWO_NEG_63, 0.0
    return SamplerPack(kind=t.distribution, l_max=t.l_max, scale=np.asarray(scale, np.float64),
                       xlo=xlo, xw=xw, flo=flo, fh=fh, eps=eps,
                       prob=alias.prob, alias=alias.alias, tail_x=float(t.x[1]))
