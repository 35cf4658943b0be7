"""Batched production fills (BASELINE.json config 4: many small requests).

The reference serves a request with a new sampler + `fill(8192)`
(`exponential.py:26-50`), paying the alias build and a kernel dispatch every
time.  Here a :class:`BatchPlan` lays many requests out back to back once
(numpy, no per-request Python objects) and `fill` runs them all in ONE launch;
request r draws samples ctr_base..ctr_base+n-1 of the counter stream of its
own seed, so each request's values equal a standalone
`UniformSource.counter(seed, ctr_base)` fill.  The plan's request table is
uploaded to a device once (`zf_batch_create`) and stays there, so every
`fill` is a single launch with no host-side table work (`zf_batch_fill`).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .tables import EXPONENTIAL, HALF_NORMAL, default_tables

REQ_DTYPE = np.dtype([("seed", "<u8"), ("ctr_base", "<u8"), ("n", "<u8"), ("out_offset", "<u8"),
                      ("dist", "<i4"), ("reserved", "<i4")])
assert REQ_DTYPE.itemsize == C.sizeof(_lib.Request)

_DIST = {"exp": _lib.EXP, "exponential": _lib.EXP, "normal": _lib.NORMAL,
         _lib.EXP: _lib.EXP, _lib.NORMAL: _lib.NORMAL}


class BatchPlan:
    """Request table + output layout (each request 16-byte aligned)."""

    def __init__(self, dists, ns, seeds, ctr_bases=None, dtype="float64"):
        import torch
        self.tdtype = torch.float64 if dtype in ("float64", torch.float64) else torch.float32
        esz = 8 if self.tdtype == torch.float64 else 4
        align = 16 // esz
        ns = np.asarray(ns, dtype=np.uint64)
        m = ns.size
        req = np.zeros(m, dtype=REQ_DTYPE)
        req["dist"] = [_DIST[d] for d in dists] if not isinstance(dists, np.ndarray) else dists
        req["n"] = ns
        req["seed"] = np.asarray(seeds, dtype=np.uint64) if m else []
        req["ctr_base"] = 0 if ctr_bases is None else np.asarray(ctr_bases, dtype=np.uint64)
        padded = (ns + np.uint64(align - 1)) // np.uint64(align) * np.uint64(align)
        offs = np.zeros(m, dtype=np.uint64)
        if m > 1:
            offs[1:] = np.cumsum(padded[:-1])
        req["out_offset"] = offs
        self.req = req
        self.offsets = offs.astype(np.int64)
        self.total = int(padded.sum()) if m else 0
        self.esz = esz
        self._resident = {}  # device index -> (tables handle, zf_batch handle)

    def _batch(self, dev):
        hit = self._resident.get(dev.index)
        if hit is None:
            tabs = _lib.device_tables(default_tables(EXPONENTIAL), default_tables(HALF_NORMAL),
                                      dev.index)
            h = C.c_void_p()
            _lib.check(_lib.lib().zf_batch_create(
                tabs.handle, self.req.ctypes.data_as(C.POINTER(_lib.Request)), self.req.size,
                _lib.F64 if self.esz == 8 else _lib.F32, C.byref(h)))
            hit = self._resident[dev.index] = (tabs, h)
        return hit[1]

    def __del__(self):
        try:
            for _, h in getattr(self, "_resident", {}).values():
                _lib.lib().zf_batch_destroy(h)
        except Exception:  # interpreter shutdown
            pass

    def fill(self, out=None, device=None):
        """One launch for every request; returns the output tensor."""
        import torch
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        if out is None:
            out = torch.empty(self.total, dtype=self.tdtype, device=dev)
        elif out.numel() < self.total or out.dtype != self.tdtype or not out.is_contiguous():
            raise ValueError("output tensor too small, wrong dtype or not contiguous")
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().zf_batch_fill(self._batch(dev), out.data_ptr(),
                                                _lib.stream_handle(dev)))
        return out

    def view(self, out, i: int):
        """Request i's samples inside a filled output tensor."""
        o, n = int(self.offsets[i]), int(self.req["n"][i])
        return out[o:o + n]


def fill_batch(requests, dtype="float64", device=None):
    """Convenience wrapper: ``requests`` = iterable of (dist, n, seed[, ctr_base]).
    One-shot (`zf_fill_batch`: the request table goes through a pinned
    staging ring, nothing stays resident).  Returns (output tensor, offsets)."""
    import torch
    reqs = list(requests)
    plan = BatchPlan([r[0] for r in reqs], [int(r[1]) for r in reqs],
                     [int(r[2]) & ((1 << 64) - 1) for r in reqs],
                     [int(r[3]) if len(r) > 3 else 0 for r in reqs], dtype=dtype)
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(plan.total, dtype=plan.tdtype, device=dev)
    tabs = _lib.device_tables(default_tables(EXPONENTIAL), default_tables(HALF_NORMAL), dev.index)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().zf_fill_batch(
            tabs.handle, plan.req.ctypes.data_as(C.POINTER(_lib.Request)), plan.req.size,
            _lib.F64 if plan.esz == 8 else _lib.F32, out.data_ptr(), _lib.stream_handle(dev)))
    return out, [int(o) for o in plan.offsets]
