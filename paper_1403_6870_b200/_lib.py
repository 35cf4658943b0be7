"""ctypes binding of the sm_100a library (include/zigfast_b200.h).

There is deliberately no CPU fallback: if `libzigfast_b200.so` is missing the
import of any sampler raises :class:`ExtensionMissing`; if there is no sm_100
device, table upload raises :class:`DeviceError`.  ctypes releases the GIL for
the duration of each call, matching the reference's `nogil=True` kernels.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib
import threading

import numpy as np

from .errors import DeviceError, ExtensionMissing

LIB_PATH = pathlib.Path(os.environ.get(
    "ZF_LIB", pathlib.Path(__file__).resolve().parent / "libzigfast_b200.so"))

# constants mirrored from the header
EXP, NORMAL = 0, 1
F64, F32 = 0, 1
GEN_XOSHIRO, GEN_SPLITMIX, GEN_REPLAY, GEN_CTR = 0, 1, 2, 3
PATH_FAST, PATH_TAIL, PATH_BOXFAST, PATH_BOXEVAL = 1, 2, 4, 8

EXPORTS = (
    "zf_abi_version", "zf_strerror", "zf_tables_create", "zf_tables_destroy", "zf_fill",
    "zf_fill_stats", "zf_stats", "zf_stats_blocks", "zf_fill_replay", "zf_fill_gid", "zf_words",
    "zf_xoshiro_jump", "zf_xoshiro_pow2_poly", "zf_fill_batch", "zf_trad_tables_create",
    "zf_format_g17", "zf_format_scratch_words", "zf_tables_create_default",
    "zf_trad_tables_create_default", "zf_batch_create", "zf_batch_fill", "zf_batch_destroy",
    "zf_batch_tables", "zf_host_register", "zf_host_unregister",
)
EXP, NORMAL, TRAD_EXP, TRAD_NORMAL = 0, 1, 2, 3

REC_DTYPE = np.dtype([("start", "<u8"), ("nwords", "<u4"), ("layer", "u1"),
                      ("path", "u1"), ("attempts", "<u2")])


class TablePack(C.Structure):
    _fields_ = [("lmax", C.c_int64), ("nslots", C.c_int64), ("sx", C.c_void_p),
                ("xlo", C.c_void_p), ("xw", C.c_void_p), ("flo", C.c_void_p),
                ("fh", C.c_void_p), ("eps", C.c_double), ("prob", C.c_void_p),
                ("alias", C.c_void_p), ("tailx", C.c_double)]


class TradPack(C.Structure):
    _fields_ = [("i_max", C.c_int64), ("se", C.c_void_p), ("kk", C.c_void_p),
                ("flo", C.c_void_p), ("fh", C.c_void_p), ("r", C.c_double)]


class Request(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("ctr_base", C.c_uint64), ("n", C.c_uint64),
                ("out_offset", C.c_uint64), ("dist", C.c_int32), ("reserved", C.c_int32)]


class StatsCfg(C.Structure):
    _fields_ = [("hist_lo", C.c_double), ("hist_hi", C.c_double), ("nbins", C.c_int32),
                ("nthresh", C.c_int32), ("abs_thresh", C.c_int32), ("moments", C.c_int32),
                ("thresh", C.c_double * 8)]


_lib = None
_lock = threading.Lock()


def lib():
    """Load the library once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ExtensionMissing(
                    f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
            L = C.CDLL(str(LIB_PATH))
            vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
            u64p = C.POINTER(C.c_uint64)
            sig = {
                "zf_abi_version": (i32, []),
                "zf_strerror": (C.c_char_p, [i32]),
                "zf_tables_create": (i32, [C.POINTER(TablePack), C.POINTER(TablePack), i32,
                                           C.POINTER(vp)]),
                "zf_tables_destroy": (i32, [vp]),
                "zf_fill": (i32, [vp, i32, i32, u64, u64, vp, u64, vp, vp]),
                "zf_fill_stats": (i32, [vp, i32, u64, u64, u64, C.POINTER(StatsCfg), vp, vp, vp]),
                "zf_stats": (i32, [i32, vp, u64, C.POINTER(StatsCfg), vp, vp, vp]),
                "zf_stats_blocks": (C.c_uint32, [u64]),
                "zf_fill_replay": (i32, [vp, i32, i32, vp, u64, u64, i32, vp, u64, vp, vp, u64p,
                                         vp]),
                "zf_fill_gid": (i32, [vp, i32, i32, i32, u64p, vp, u64, vp, u64, vp, vp, vp]),
                "zf_words": (i32, [i32, u64p, u64, vp, vp]),
                "zf_xoshiro_jump": (i32, [u64p, u64]),
                "zf_xoshiro_pow2_poly": (i32, [i32, u64p]),
                "zf_fill_batch": (i32, [vp, C.POINTER(Request), i32, i32, vp, vp]),
                "zf_trad_tables_create": (i32, [C.POINTER(TradPack), C.POINTER(TradPack), i32,
                                                C.POINTER(vp)]),
                "zf_format_g17": (i32, [vp, u64, vp, u64, vp, vp]),
                "zf_format_scratch_words": (u64, [u64]),
                "zf_tables_create_default": (i32, [i32, C.POINTER(vp)]),
                "zf_trad_tables_create_default": (i32, [i32, C.POINTER(vp)]),
                "zf_batch_create": (i32, [vp, C.POINTER(Request), i32, i32, C.POINTER(vp)]),
                "zf_batch_fill": (i32, [vp, vp, vp]),
                "zf_batch_destroy": (i32, [vp]),
                "zf_batch_tables": (vp, [vp]),
                "zf_host_register": (i32, [vp, u64]),
                "zf_host_unregister": (i32, [vp]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype, fn.argtypes = res, args
            if L.zf_abi_version() != 1:
                raise ExtensionMissing("libzigfast_b200.so ABI version mismatch; rebuild")
            _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise DeviceError(status, lib().zf_strerror(status).decode())


def u64p(arr: np.ndarray):
    assert arr.dtype == np.uint64 and arr.flags.c_contiguous
    return arr.ctypes.data_as(C.POINTER(C.c_uint64))


def stream_handle(device) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


class DeviceTables:
    """The uploaded pair of packs (exp + half-normal) on one device."""

    def __init__(self, exp_pack, hn_pack, device_index: int):
        self._keep = []
        packs = [self._cpack(exp_pack), self._cpack(hn_pack)]
        handle = C.c_void_p()
        check(lib().zf_tables_create(C.byref(packs[0]), C.byref(packs[1]), device_index,
                                     C.byref(handle)))
        self.handle = handle
        self.device_index = device_index

    def _cpack(self, p) -> TablePack:
        arrays = {k: np.ascontiguousarray(getattr(p, k), dtype=np.float64)
                  for k in ("scale", "xlo", "xw", "flo", "fh", "prob")}
        alias = np.ascontiguousarray(p.alias, dtype=np.int64)
        self._keep.extend(arrays.values())
        self._keep.append(alias)
        ptr = {k: v.ctypes.data for k, v in arrays.items()}
        return TablePack(p.l_max, p.l_max + 1, ptr["scale"], ptr["xlo"], ptr["xw"], ptr["flo"],
                         ptr["fh"], p.eps, ptr["prob"], alias.ctypes.data, p.tail_x)

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.zf_tables_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass


class DeviceTradTables(DeviceTables):
    """The uploaded traditional packs (exp + half-normal) on one device."""

    def __init__(self, exp_pack, hn_pack, device_index: int):
        self._keep = []
        packs = [self._tpack(exp_pack), self._tpack(hn_pack)]
        handle = C.c_void_p()
        check(lib().zf_trad_tables_create(C.byref(packs[0]), C.byref(packs[1]), device_index,
                                          C.byref(handle)))
        self.handle = handle
        self.device_index = device_index

    def _tpack(self, p) -> TradPack:
        se, flo, fh = (np.ascontiguousarray(a, dtype=np.float64) for a in (p.se, p.flo, p.fh))
        kk = np.ascontiguousarray(p.kk, dtype=np.uint64)
        self._keep.extend((se, flo, fh, kk))
        return TradPack(se.size, se.ctypes.data, kk.ctypes.data, flo.ctypes.data,
                        fh.ctypes.data, p.r)


_tables_cache: dict = {}
_tables_lock = threading.Lock()


def _cached_upload(key, exp_tables, hn_tables, make):
    """One upload per (tables pair, device), shared by every sampler and host
    thread (the handle is immutable and thread-safe)."""
    with _tables_lock:
        hit = _tables_cache.get(key)
        if hit is None or hit[0] is not exp_tables or hit[1] is not hn_tables:
            hit = (exp_tables, hn_tables, make())
            _tables_cache[key] = hit
        return hit[2]


def device_tables(exp_tables, hn_tables, device_index: int) -> DeviceTables:
    """Cached upload of a (exp, half-normal) table pair to a device."""
    from .tables import make_pack
    return _cached_upload((id(exp_tables), id(hn_tables), device_index), exp_tables, hn_tables,
                          lambda: DeviceTables(make_pack(exp_tables), make_pack(hn_tables),
                                               device_index))


def device_trad_tables(exp_tables, hn_tables, device_index: int) -> DeviceTradTables:
    """Cached upload of a traditional (exp, half-normal) table pair."""
    from .traditional import trad_pack
    return _cached_upload(("trad", id(exp_tables), id(hn_tables), device_index), exp_tables,
                          hn_tables, lambda: DeviceTradTables(trad_pack(exp_tables),
                                                              trad_pack(hn_tables), device_index))
