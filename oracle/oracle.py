"""CPU ORACLE (ctypes front end of oracle/zf_oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
`--impl reference` arm) may import this module.  The product package never does.

Everything here is independent of the product's host code on purpose: the
tables are parsed from the shipped ZIGT files with a separate reader, the
overhang arrays follow `_packs.py:15-28` directly, and the alias arrays come
from the C restatement of `alias.py:32-63`, so a product-side mistake in any
of those cannot cancel against the checker.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib
import struct
import subprocess
import zlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libzf_oracle.so"
DATA = HERE.parent / "paper_1403_6870_b200" / "data"

SRC_XOSHIRO, SRC_SPLITMIX, SRC_REPLAY, SRC_CTR = 0, 1, 2, 3
EXP, NORMAL, TRAD_EXP, TRAD_NORMAL = 0, 1, 2, 3

REC_DTYPE = np.dtype([("start", "<u8"), ("nwords", "<u4"), ("layer", "u1"),
                      ("path", "u1"), ("attempts", "<u2")])
P_FAST, P_TAIL, P_BOXFAST, P_BOXEVAL = 1, 2, 4, 8


def build() -> pathlib.Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        u64p = C.POINTER(C.c_uint64)
        L.orc_fill.restype = C.c_uint64
        L.orc_fill.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, u64p, u64p, C.c_uint64,
                               C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_fill_ctr.restype = None
        L.orc_fill_ctr.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                   C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_ctr_words.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.orc_words.argtypes = [C.c_int, u64p, C.c_uint64, u64p]
        L.orc_seed_xoshiro.argtypes = [C.c_uint64, u64p]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_build_alias_vose.restype = C.c_int
        L.orc_build_alias_vose.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_aggregate.restype = C.c_double
        L.orc_aggregate.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, u64p, C.c_uint64]
        L.orc_fill_sharded_chunked.restype = C.c_int
        L.orc_fill_sharded_chunked.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                               C.c_uint64, C.c_int, C.c_uint64,
                                               C.POINTER(C.c_double)]
        L.orc_check_ctr.restype = C.c_int64
        L.orc_check_ctr.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                    C.c_void_p, C.c_int, C.c_uint64, C.c_int, u64p]
        L.orc_count_ctr.restype = C.c_int
        L.orc_count_ctr.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                    C.c_uint64, C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int,
                                    u64p]
        L.orc_fill_sharded.restype = C.c_int
        L.orc_fill_sharded.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                       C.c_uint64, C.c_int]
        dp = C.POINTER(C.c_double)
        L.orc_trad_solve.restype = C.c_int
        L.orc_trad_solve.argtypes = [C.c_int, C.c_int, dp, dp, dp, dp, dp]
        L.orc_trad_pack_arrays.restype = None
        L.orc_trad_pack_arrays.argtypes = [C.c_int, C.c_int, dp, dp, dp, C.c_double, C.c_double,
                                           dp, u64p, dp, dp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# --- independent table reader (ZIGT: zigfast/tableio.py:97-143) -------------

def read_zigt(kind: str):
    blob = (DATA / f"{kind}_256.zigt").read_bytes()
    body, crc = blob[:-4], struct.unpack("<I", blob[-4:])[0]
    assert zlib.crc32(body) == crc, "ZIGT checksum"
    magic, ver, code, i_max, l_max = struct.unpack_from("<4sBBII", body, 0)
    assert magic == b"ZIGT" and ver == 1
    total_mass, eps = struct.unpack_from("<2d", body, 14)
    n = l_max + 1
    x, f, a = (np.frombuffer(body, "<f8", n, 30 + 8 * n * k).copy() for k in range(3))
    return dict(l_max=l_max, i_max=i_max, eps=eps, x=x, f=f, a=a, total_mass=total_mass)


class Pack(C.Structure):
    _fields_ = [("lmax", C.c_int64), ("nslots", C.c_int64), ("sx", C.c_void_p),
                ("xlo", C.c_void_p), ("xw", C.c_void_p), ("flo", C.c_void_p),
                ("fh", C.c_void_p), ("eps", C.c_double), ("prob", C.c_void_p),
                ("alias", C.c_void_p), ("tailx", C.c_double)]


class OraclePack:
    """Flat pack for one density; keeps its numpy arrays alive."""

    def __init__(self, kind: str):
        t = read_zigt(kind)
        n = t["l_max"] + 1
        xe = np.append(t["x"], 0.0)
        fe = np.append(t["f"], 1.0)
        self.xlo, self.xw, self.flo, self.fh = (np.zeros(n) for _ in range(4))
        for j in range(1, n):                      # _packs.py:20-25
            self.xlo[j] = xe[j + 1]
            self.xw[j] = xe[j] - xe[j + 1]
            self.flo[j] = fe[j]
            self.fh[j] = fe[j + 1] - fe[j]
        if kind == "exponential":
            self.sx = t["x"] * 2.0 ** -64
            eps = t["eps"]
        else:
            self.sx = t["x"] * 2.0 ** -63
            eps = 0.0
        self.prob = np.empty(n)
        self.alias = np.empty(n, dtype=np.int64)
        rc = lib().orc_build_alias_vose(_ptr(np.ascontiguousarray(t["a"])), n, _ptr(self.prob),
                                        _ptr(self.alias))
        assert rc == 0
        self.tables = t
        self.c = Pack(t["l_max"], n, _ptr(self.sx).value, _ptr(self.xlo).value,
                      _ptr(self.xw).value, _ptr(self.flo).value, _ptr(self.fh).value, eps,
                      _ptr(self.prob).value, _ptr(self.alias).value, float(t["x"][1]))


class TradPack(C.Structure):
    _fields_ = [("i_max", C.c_int64), ("se", C.c_void_p), ("kk", C.c_void_p),
                ("flo", C.c_void_p), ("fh", C.c_void_p), ("r", C.c_double)]


class OracleTradPack:
    """Traditional tables solved by the C restatement of solve_traditional
    (traditional.py:56-96) and packed like traditional._pack (:113-121)."""

    def __init__(self, kind: str, i_max: int = 256):
        code = 0 if kind == "exponential" else 1
        dp = C.POINTER(C.c_double)
        self.x, self.f, self.k = (np.empty(i_max) for _ in range(3))
        r, v = C.c_double(), C.c_double()
        rc = lib().orc_trad_solve(code, i_max, self.x.ctypes.data_as(dp),
                                  self.f.ctypes.data_as(dp), self.k.ctypes.data_as(dp),
                                  C.byref(r), C.byref(v))
        assert rc == 0, rc
        self.r, self.v = r.value, v.value
        self.se, self.flo, self.fh = (np.empty(i_max) for _ in range(3))
        self.kk = np.empty(i_max, dtype=np.uint64)
        lib().orc_trad_pack_arrays(code, i_max, self.x.ctypes.data_as(dp),
                                   self.f.ctypes.data_as(dp), self.k.ctypes.data_as(dp),
                                   self.r, self.v, self.se.ctypes.data_as(dp), _u64p(self.kk),
                                   self.flo.ctypes.data_as(dp), self.fh.ctypes.data_as(dp))
        self.c = TradPack(i_max, _ptr(self.se).value, _ptr(self.kk).value, _ptr(self.flo).value,
                          _ptr(self.fh).value, self.r)


_packs = {}


def packs(dist=EXP):
    """(h, e) pack pair for a distribution code (modified or traditional)."""
    if _dist(dist) in (TRAD_EXP, TRAD_NORMAL):
        if "texp" not in _packs:
            _packs["texp"] = OracleTradPack("exponential")
            _packs["thn"] = OracleTradPack("halfnormal")
        return _packs["thn"], _packs["texp"]
    if "exp" not in _packs:
        _packs["exp"] = OraclePack("exponential")
        _packs["hn"] = OraclePack("halfnormal")
    return _packs["hn"], _packs["exp"]


def _dist(dist) -> int:
    return {"exp": EXP, "exponential": EXP, "normal": NORMAL, "trad_exp": TRAD_EXP,
            "trad_normal": TRAD_NORMAL, EXP: EXP, NORMAL: NORMAL, TRAD_EXP: TRAD_EXP,
            TRAD_NORMAL: TRAD_NORMAL}[dist]


# --- word streams -------------------------------------------------------------

def xoshiro_state(seed: int) -> np.ndarray:
    st = np.zeros(4, dtype=np.uint64)
    lib().orc_seed_xoshiro(seed & (2**64 - 1), _u64p(st))
    return st


def words(generator: str, seed: int, n: int) -> np.ndarray:
    if generator == "xoshiro256++":
        st, kind = xoshiro_state(seed), SRC_XOSHIRO
    else:
        st, kind = np.array([seed & (2**64 - 1)], dtype=np.uint64), SRC_SPLITMIX
    out = np.empty(n, dtype=np.uint64)
    lib().orc_words(kind, _u64p(st), n, _u64p(out))
    return out


def derive_seed(base: int, stream: int) -> int:
    return int(lib().orc_derive_seed(base & (2**64 - 1), stream))


# --- fills ----------------------------------------------------------------------

def fill_stream(dist, n: int, *, generator="xoshiro256++", seed=0, replay_words=None,
                cursor=0, records=False):
    """Reference fill over a sequential stream; returns (values, counters, recs, used)."""
    h, e = packs(dist)
    out = np.empty(n, dtype=np.float64)
    cnt = np.zeros(6, dtype=np.int64)
    recs = np.zeros(n, dtype=REC_DTYPE) if records else None
    wbuf = None
    if replay_words is not None:
        wbuf = np.ascontiguousarray(replay_words, dtype=np.uint64)
        st, kind = np.array([cursor], dtype=np.uint64), SRC_REPLAY
    elif generator == "xoshiro256++":
        st, kind = xoshiro_state(seed), SRC_XOSHIRO
    else:
        st, kind = np.array([seed & (2**64 - 1)], dtype=np.uint64), SRC_SPLITMIX
    used = lib().orc_fill(_dist(dist), C.byref(h.c), C.byref(e.c), kind, _u64p(st),
                          _u64p(wbuf) if wbuf is not None else None,
                          0 if wbuf is None else wbuf.size, _ptr(out), n, _ptr(cnt),
                          _ptr(recs) if recs is not None else None)
    return out, cnt, recs, int(used)


def fill_ctr(dist, n: int, seed: int, ctr_base: int = 0, records=False):
    """Production ("ctr") stream restated on the CPU; returns (values, counters, recs)."""
    h, e = packs(dist)
    out = np.empty(n, dtype=np.float64)
    cnt = np.zeros(6, dtype=np.int64)
    recs = np.zeros(n, dtype=REC_DTYPE) if records else None
    lib().orc_fill_ctr(_dist(dist), C.byref(h.c), C.byref(e.c), seed & (2**64 - 1), ctr_base,
                       _ptr(out), n, _ptr(cnt), _ptr(recs) if recs is not None else None)
    return out, cnt, recs


def check_ctr(dist, got: np.ndarray, seed: int, ctr_base: int = 0,
              threads: int | None = None) -> tuple[int, int]:
    """Compare EVERY sample of a production fill (float64 or float32, C-contiguous)
    with the oracle, in place and on `threads` host threads (default: all of
    them).  Returns (number of mismatching samples, lowest mismatching index or
    len(got))."""
    if got.dtype not in (np.float64, np.float32) or not got.flags.c_contiguous:
        raise ValueError("check_ctr needs a contiguous float64/float32 array")
    h, e = packs(dist)
    threads = threads or len(os.sched_getaffinity(0))
    first = C.c_uint64()
    bad = lib().orc_check_ctr(_dist(dist), C.byref(h.c), C.byref(e.c), seed & (2**64 - 1),
                              ctr_base, _ptr(got), int(got.dtype == np.float32), got.size,
                              threads, C.byref(first))
    assert bad >= 0
    return int(bad), int(first.value)


def count_ctr(dist, n: int, seed: int, ctr_base: int = 0, thresholds=(), abs_thresh=False,
              threads: int | None = None) -> list[int]:
    """Counts of x > t (|x| > t) over `n` production draws, nothing stored
    (config 5's generate-and-count), on `threads` host threads."""
    h, e = packs(dist)
    threads = threads or len(os.sched_getaffinity(0))
    t = np.asarray(thresholds, dtype=np.float64)
    counts = np.zeros(max(len(t), 1), dtype=np.uint64)
    rc = lib().orc_count_ctr(_dist(dist), C.byref(h.c), C.byref(e.c), seed & (2**64 - 1),
                             ctr_base, n, t.ctypes.data_as(C.POINTER(C.c_double)), len(t),
                             int(abs_thresh), threads, _u64p(counts))
    assert rc == 0
    return [int(c) for c in counts[:len(t)]]


def ctr_words(seed: int, K: int, m: int) -> np.ndarray:
    out = np.empty(m, dtype=np.uint64)
    lib().orc_ctr_words(seed & (2**64 - 1), K, m, _u64p(out))
    return out


def aggregate(dist, n: int, seed: int) -> float:
    h, e = packs(dist)
    st = xoshiro_state(seed)
    return float(lib().orc_aggregate(_dist(dist), C.byref(h.c), C.byref(e.c), SRC_XOSHIRO,
                                     _u64p(st), n))


def fill_sharded(dist, n: int, seed: int, threads: int | None = None,
                 out: np.ndarray | None = None) -> np.ndarray:
    """The reference's --jobs sharding (quality.py:121-126) on `threads` host threads."""
    h, e = packs(dist)
    threads = threads or len(os.sched_getaffinity(0))
    out = np.empty(n, dtype=np.float64) if out is None else out
    rc = lib().orc_fill_sharded(_dist(dist), C.byref(h.c), C.byref(e.c), seed & (2**64 - 1),
                                _ptr(out), n, threads)
    assert rc == 0
    return out


def fill_sharded_chunked(dist, n: int, seed: int, threads: int | None = None,
                         chunk: int = 1 << 20) -> float:
    """`fill_sharded` through one reused `chunk`-sample buffer per thread (the
    reference's run_quality fill pattern); returns a checksum."""
    h, e = packs(dist)
    threads = threads or len(os.sched_getaffinity(0))
    cs = C.c_double()
    rc = lib().orc_fill_sharded_chunked(_dist(dist), C.byref(h.c), C.byref(e.c),
                                        seed & (2**64 - 1), n, threads, chunk, C.byref(cs))
    assert rc == 0
    return cs.value
