"""ExpSampler / NormalSampler: the reference's sampling API on B200.

Mirrors `zigfast/exponential.py:23-88` and `zigfast/normal.py:21-88`: same
constructors, `sample`, `fill`, `fill_counted`, `aggregate`, `path_counts`,
`reset_counters`, `overhang_attempt`, `tail_start`.  Every draw runs in the
sm_100a library; the generator id of the source picks the kernel path:

* ``UniformSource(seed, "ctr")`` -- production mode: one asynchronous launch
  of the counter-stream kernel (`zf_fill`).
* xoshiro256++ / splitmix64 / replay -- oracle mode: the reference's exact
  sequential stream, generated and resolved in parallel on the GPU
  (`zf_fill_gid`), host state advanced exactly as the reference's kernel
  advances `state` in place.

`fill(out)` accepts an int (returns a new CUDA float64 tensor), a CUDA tensor
(float64 / float32, filled in place), or a host numpy array / CPU tensor
(filled through the device, chunked, returned as the same object).
"""

from __future__ import annotations

import contextlib
import math
import threading
import weakref
from collections import OrderedDict

import numpy as np

from . import _lib
from .errors import ZigfastError
from .tables import (EXPONENTIAL, HALF_NORMAL, ZigguratTables, build_alias, default_tables)
from .uniform import CTR_LIMIT, UniformSource

_HOST_CHUNK = 1 << 24  # samples per device chunk when the destination is host memory
_STAGE_BYTES = 64 << 20  # bytes per pinned staging chunk (pageable host destinations)
_STAGE_MIN_BYTES = 1 << 20  # smaller pageable fills copy directly


class _Staging:
    """Two pinned host buffers + two device buffers + a copy stream, kept per
    device (pinning 128 MB costs more than the fill it serves)."""

    def __init__(self, device):
        import torch
        self.stream = torch.cuda.Stream(device)
        self._host = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True)
                      for _ in range(2)]
        self._dev = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, device=device)
                     for _ in range(2)]
        self.samples = 0

    def host_bufs(self, dtype):
        return [b.view(dtype) for b in self._host]

    def device_bufs(self, dtype):
        return [b.view(dtype) for b in self._dev]


_stage_cache: dict = {}
_stage_lock = threading.Lock()

# -- page-locking of caller-owned host arrays ------------------------------------
# A pageable destination of >= _REGISTER_MIN_BYTES is page-locked in place
# (cudaHostRegister) once and kept registered while the array lives (a weakref
# finalizer unregisters it before numpy frees the memory), so the device DMAs
# straight into it at the link rate; repeated fills of the same buffer -- the
# reference's `fill(out)` pattern -- pay the ~30 ms/GiB registration once.
# At most _REGISTER_CAP bytes stay registered (least recently used evicted).
_REGISTER_MIN_BYTES = 64 << 20
_REGISTER_CAP = 64 << 30
_reg_lock = threading.Lock()
_registered: "OrderedDict[int, tuple[int, object]]" = OrderedDict()


def _unregister(ptr: int) -> None:
    with _reg_lock:
        entry = _registered.pop(ptr, None)
    if entry is not None:
        try:
            _lib.lib().zf_host_unregister(ptr)
        except Exception:  # interpreter shutdown
            pass


def _owner(arr: np.ndarray):
    """The ndarray that owns ``arr``'s memory (following view bases), or None."""
    b = arr
    while isinstance(b.base, np.ndarray):
        b = b.base
    return b if b.base is None and b.flags.owndata else None


def _page_locked(arr) -> bool:
    """Register ``arr``'s owning buffer with the driver (cached); False if it
    cannot be (not a plain numpy allocation, too small, or refused)."""
    if not isinstance(arr, np.ndarray) or arr.nbytes < _REGISTER_MIN_BYTES:
        return False
    owner = _owner(arr)
    if owner is None:
        return False
    ptr, nbytes = owner.ctypes.data, owner.nbytes
    evict = []
    with _reg_lock:
        hit = _registered.get(ptr)
        if hit is not None and hit[0] == nbytes:
            _registered.move_to_end(ptr)
            return True
        total = sum(v[0] for v in _registered.values()) + nbytes
        for p, (nb, fin) in _registered.items():
            if total <= _REGISTER_CAP:
                break
            evict.append((p, fin))
            total -= nb
    for p, fin in evict:
        fin.detach()
        _unregister(p)
    if _lib.lib().zf_host_register(ptr, nbytes) != 0:
        return False  # e.g. another thread registered it first: stage instead
    with _reg_lock:
        _registered[ptr] = (nbytes, weakref.finalize(owner, _unregister, ptr))
    return True


@contextlib.contextmanager
def _staging(device, element_size: int):
    """The device's cached staging set, or a private one while another thread
    holds it."""
    with _stage_lock:
        entry = _stage_cache.get(device.index)
        if entry is None:
            entry = _stage_cache[device.index] = (_Staging(device), threading.Lock())
    stage, lock = entry
    if not lock.acquire(blocking=False):
        stage, lock = _Staging(device), None
    try:
        stage.samples = _STAGE_BYTES // element_size
        yield stage
    finally:
        if lock is not None:
            lock.release()


class PathCounts:
    """Per-path hit counts (`_packs.py:67-93`); slots as `_kernels.py:23-27`."""

    __slots__ = ("byte_draws", "common", "overhang_fast", "band_evals", "tail", "box_attempts")

    def __init__(self, *vals):
        for k, v in zip(self.__slots__, vals):
            setattr(self, k, int(v))

    @classmethod
    def from_array(cls, arr) -> "PathCounts":
        return cls(*(int(v) for v in arr))

    def as_tuple(self):
        return tuple(getattr(self, k) for k in self.__slots__)

    def __eq__(self, other):
        return isinstance(other, PathCounts) and self.as_tuple() == other.as_tuple()

    def __repr__(self):
        return "PathCounts(" + ", ".join(f"{k}={getattr(self, k)}" for k in self.__slots__) + ")"

    @property
    def common_fraction(self) -> float:
        return self.common / self.byte_draws if self.byte_draws else 0.0

    @property
    def tail_fraction(self) -> float:
        return self.tail / self.byte_draws if self.byte_draws else 0.0

    @property
    def band_eval_fraction(self) -> float:
        return self.band_evals / self.box_attempts if self.box_attempts else 0.0


_ALIAS_CACHE: dict = {}


def _alias_for(tables: ZigguratTables):
    """The alias table of immutable `tables`, built once per tables object (the
    reference rebuilds it per sampler, exponential.py:33; same arrays)."""
    hit = _ALIAS_CACHE.get(id(tables))
    if hit is None or hit[0] is not tables:
        hit = (tables, build_alias(tables.a))
        _ALIAS_CACHE[id(tables)] = hit
    return hit[1]


class _SamplerBase:
    """Device, source, counters and the fill/launch plumbing shared by the
    modified samplers and the traditional baseline (`traditional.py`)."""

    _dist: int
    _dev_tables: "_lib.DeviceTables"

    def _init_device(self, source, device) -> None:
        import torch
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise ValueError("samplers run on CUDA devices only (no CPU fallback)")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.source = source if source is not None else UniformSource()
        self._counters = torch.zeros(6, dtype=torch.int64, device=self.device)

    # -- counters ---------------------------------------------------------------
    @property
    def counters(self) -> np.ndarray:
        return self._counters.cpu().numpy()

    @property
    def path_counts(self) -> PathCounts:
        return PathCounts.from_array(self.counters)

    def reset_counters(self) -> None:
        self._counters.zero_()

    # -- core launch --------------------------------------------------------------
    def _launch(self, dst, counted: bool, recs=None) -> None:
        """Fill the contiguous CUDA tensor ``dst`` from the source, advancing it."""
        import torch
        n = dst.numel()
        if n == 0:
            return
        dtype = {torch.float64: _lib.F64, torch.float32: _lib.F32}.get(dst.dtype)
        if dtype is None:
            raise TypeError(f"output dtype must be float64 or float32, got {dst.dtype}")
        if not dst.is_contiguous():
            raise ValueError("output tensor must be contiguous")
        src = self.source
        if src.gid == _lib.GEN_CTR and int(src.state[1]) + n > CTR_LIMIT:
            raise ValueError("counter stream exhausted (2^44 samples per seed)")
        words_ptr, nwords = None, 0
        if src.gid == _lib.GEN_REPLAY:
            w = src.replay_words_device(self.device)
            words_ptr, nwords = w.data_ptr(), w.numel()
        cnt = self._counters.data_ptr() if counted else None
        rec_ptr = recs.data_ptr() if recs is not None else None
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().zf_fill_gid(
                self._dev_tables.handle, self._dist, dtype, src.gid, _lib.u64p(src.state),
                words_ptr, nwords, dst.data_ptr(), n, rec_ptr, cnt,
                _lib.stream_handle(self.device)))

    def _fill(self, out, counted: bool):
        import torch
        if isinstance(out, (int, np.integer)):
            if out < 0:
                raise ValueError("size must be nonnegative")
            dst = torch.empty(int(out), dtype=torch.float64, device=self.device)
            self._launch(dst, counted)
            return dst
        if isinstance(out, torch.Tensor) and out.is_cuda:
            if out.device != self.device:
                raise ValueError(f"output on {out.device}, sampler on {self.device}")
            if out.is_contiguous():
                self._launch(out.view(-1), counted)
            else:
                # a strided view (the reference's kernels index out[k] through any
                # strides): draw into a dense buffer, scatter in element order
                tmp = torch.empty(out.shape, dtype=out.dtype, device=self.device)
                self._launch(tmp.view(-1), counted)
                out.copy_(tmp)
            return out
        # host destination: numpy array or CPU tensor -> through the device in chunks
        if isinstance(out, np.ndarray) and out.flags.c_contiguous:
            _page_locked(out)  # large pageable arrays: DMA in place from now on
        host = torch.from_numpy(out) if isinstance(out, np.ndarray) else out
        if not isinstance(host, torch.Tensor) or host.is_cuda:
            raise TypeError("out must be an int, a CUDA tensor, a numpy array or a CPU tensor")
        if not host.is_contiguous():
            # strided host views work in the reference (numba indexes out[k]):
            # fill a dense array, then assign in element order
            dense = torch.empty(host.shape, dtype=host.dtype)
            self._fill_host(dense.view(-1), counted)
            host.copy_(dense)
            return out
        self._fill_host(host.view(-1), counted)
        return out

    def _fill_host(self, host, counted: bool) -> None:
        """Device fill + D2H copy, double-buffered so chunk i+1 generates while
        chunk i copies (the copy engine is the bound for host destinations).
        Pageable destinations (a plain numpy array, the reference's usage) of
        64 MiB or more are page-locked in place and then DMA'd like pinned
        memory (`_page_locked`); smaller or unregistrable ones go through
        pinned staging buffers: the driver's own pageable D2H path runs at
        ~20 GB/s on the B200 box, a pinned copy at ~57 GB/s plus a
        multi-threaded host memcpy at ~45 GB/s, overlapped chunk by chunk."""
        import torch
        n = host.numel()
        if n == 0:
            return
        if not host.is_pinned() and n * host.element_size() >= _STAGE_MIN_BYTES:
            with _staging(self.device, host.element_size()) as stage:
                self._fill_staged(host, counted, stage)
            return
        chunk = min(n, _HOST_CHUNK)
        bufs = [torch.empty(chunk, dtype=host.dtype, device=self.device) for _ in range(2)]
        copy_stream = torch.cuda.Stream(self.device)
        compute = torch.cuda.current_stream(self.device)
        done = [None, None]
        for i, off in enumerate(range(0, n, chunk)):
            m = min(chunk, n - off)
            b = i & 1
            if done[b] is not None:
                compute.wait_event(done[b])  # buffer b's previous copy finished
            self._launch(bufs[b][:m], counted)
            ready = torch.cuda.Event()
            ready.record(compute)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(ready)
                host[off:off + m].copy_(bufs[b][:m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                done[b] = ev
        copy_stream.synchronize()

    def _fill_staged(self, host, counted: bool, stage) -> None:
        """Pageable host destination: generate chunk i on the device, copy it
        D2H into pinned buffer i%2 on a side stream, and copy pinned buffer
        (i-1)%2 into the destination on the host meanwhile."""
        import torch
        n = host.numel()
        chunk = stage.samples
        dev, pinned = stage.device_bufs(host.dtype), stage.host_bufs(host.dtype)
        copy_stream = stage.stream
        compute = torch.cuda.current_stream(self.device)
        pending = []  # (event, pinned slot, destination offset, count)
        freed = [None, None]  # device buffer b may be refilled after this event

        def drain_one():
            ev, b, off, m = pending.pop(0)
            ev.synchronize()
            host[off:off + m].copy_(pinned[b][:m])

        for i, off in enumerate(range(0, n, chunk)):
            m = min(chunk, n - off)
            b = i & 1
            if len(pending) == 2:
                drain_one()  # pinned slot b is about to be overwritten
            if freed[b] is not None:
                compute.wait_event(freed[b])
            self._launch(dev[b][:m], counted)
            ready = torch.cuda.Event()
            ready.record(compute)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(ready)
                pinned[b][:m].copy_(dev[b][:m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
            freed[b] = ev
            pending.append((ev, b, off, m))
        while pending:
            drain_one()

    # -- reference API -------------------------------------------------------------
    _SAMPLE_BLOCK = 4096

    def sample(self) -> float:
        """One draw.  Production sources serve scalar draws from a block of
        the next ``_SAMPLE_BLOCK`` values of their counter stream (one launch and
        one copy per block); the source still advances by exactly one sample per
        call, so interleaved fill() / sample() calls see the same stream as
        repeated sample() calls.  Sequential (oracle-mode) sources do the same
        with per-draw word counts (`_sample_sequential`)."""
        src = self.source
        if src.gid != _lib.GEN_CTR:
            return self._sample_sequential(src)
        seed, ctr = int(src.state[0]), int(src.state[1])
        cache = getattr(self, "_scalar_cache", None)
        if cache is None or cache[0] != seed or not cache[1] <= ctr < cache[1] + len(cache[2]):
            m = min(self._SAMPLE_BLOCK, CTR_LIMIT - ctr)
            if m <= 0:
                raise ValueError("counter stream exhausted (2^44 samples per seed)")
            self.source = UniformSource.counter(seed, ctr)  # a throwaway copy
            try:
                cache = (seed, ctr, self._fill(m, False).cpu().numpy())
            finally:
                self.source = src
            self._scalar_cache = cache
        src.state[1] = np.uint64(ctr + 1)
        return float(cache[2][ctr - cache[1]])

    def _sample_sequential(self, src) -> float:
        """Scalar draw from a sequential (reference) stream.  A block of the next
        ``_SAMPLE_BLOCK`` draws and their word counts is resolved once on a
        clone of the source; each call then returns the next value and advances
        the real source by exactly that draw's words, as the reference's
        `sample()` does.  Any outside change of the source state invalidates
        the block; a block that cannot be resolved (a replay list on which some
        later draw never finishes) falls back to one draw per call."""
        k = 4 if src.gid == _lib.GEN_XOSHIRO else 1
        c = getattr(self, "_seq_cache", None)
        valid = (c is not None and c["src"] is src and c["state"] is src.state
                 and c["i"] < len(c["vals"]) and np.array_equal(c["expect"], src.state[:k]))
        if not valid:
            self.source = src.clone()  # resolve the block on a throwaway copy
            try:
                vals, recs = self.fill_records(self._SAMPLE_BLOCK)
            except ZigfastError:
                vals = None
            finally:
                self.source = src
            if vals is None:  # fall back to one draw on the real source
                return float(self._fill(1, False).item())
            c = {"src": src, "state": src.state, "vals": vals.cpu().numpy(),
                 "nw": recs["nwords"].astype(np.int64), "i": 0}
            self._seq_cache = c
        i = c["i"]
        src.jump(int(c["nw"][i]))
        c["i"] = i + 1
        c["expect"] = src.state[:k].copy()
        return float(c["vals"][i])

    def sample_counted(self) -> float:
        return float(self._fill(1, True).item())

    def fill(self, out):
        """Fill ``out`` (or a fresh length-``out`` CUDA buffer) with draws."""
        return self._fill(out, False)

    def fill_counted(self, out):
        return self._fill(out, True)

    def fill_records(self, n: int):
        """Oracle mode only: values plus per-sample path records (zf_path_rec)."""
        import torch
        if self.source.gid == _lib.GEN_CTR:
            raise ValueError("path records need a sequential (oracle-mode) source")
        out = torch.empty(n, dtype=torch.float64, device=self.device)
        recs = torch.empty(n * _lib.REC_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        self._launch(out, False, recs=recs)
        return out, recs.cpu().numpy().view(_lib.REC_DTYPE)

    def aggregate(self, n: int) -> float:
        """Sum of ``n`` fresh draws (the reference's bench loop).

        Production sources use the fused generate-and-reduce kernel (nothing is
        written to HBM); sequential sources fill a device buffer and reduce it.
        The sum is exact-merged across blocks (fsum), so it differs from the
        reference's left-to-right float sum only by that sum's own rounding.
        """
        from .quality import device_sums
        import torch
        if n <= 0:
            return 0.0
        src = self.source
        if src.gid == _lib.GEN_CTR:
            sums, _ = device_sums(self, n, moments=1)
            return sums[0]
        total = []
        left = n
        while left:
            m = min(left, _HOST_CHUNK)
            buf = torch.empty(m, dtype=torch.float64, device=self.device)
            self._launch(buf, False)
            from .quality import buffer_sums
            total.append(buffer_sums(buf, moments=1)[0][0])
            left -= m
        return math.fsum(total)


class _Sampler(_SamplerBase):
    """Modified-ziggurat sampler state: tables, alias, uploaded packs."""

    def __init__(self, tables, exp_tables, source, device):
        self._init_device(source, device)
        self.tables = tables
        self.exp_tables = exp_tables
        self.alias = _alias_for(tables)
        hn = tables if tables.distribution == HALF_NORMAL else default_tables(HALF_NORMAL)
        self._dev_tables = _lib.device_tables(exp_tables, hn, self.device.index)


class ExpSampler(_Sampler):
    """Exponential(1) sampler (`exponential.py:23-88`)."""

    _dist = _lib.EXP

    def __init__(self, tables: ZigguratTables | None = None, source: UniformSource | None = None,
                 device=None):
        if tables is None:
            tables = default_tables(EXPONENTIAL)
        if tables.distribution != EXPONENTIAL:
            raise ValueError(f"need exponential tables, got {tables.distribution!r}")
        super().__init__(tables, tables, source, device)

    def overhang_attempt(self, j: int, ux: float, uy: float):
        """One bounded-box attempt from explicit coordinates (host probe,
        same arithmetic as the device body); ``(accepted, x, evaluated)``."""
        if not 1 <= j <= self.tables.l_max:
            raise IndexError(f"bounded slot out of range: {j}")
        xl, xr, fb, ft = self.tables.box_bounds(j)
        xw, fh, eps = xr - xl, ft - fb, float(self.tables.epsilon_max)
        if ux > 1.0 - uy:
            ux, uy = 1.0 - uy, 1.0 - ux
        if uy < 1.0 - ux - eps:
            return True, xl + ux * xw, False
        x = xl + ux * xw
        if fb + uy * fh < np.exp(-x):
            return True, x, True
        return False, None, True


class NormalSampler(_Sampler):
    """N(0,1) sampler: half-normal magnitude + sign (`normal.py:21-88`)."""

    _dist = _lib.NORMAL

    def __init__(self, tables: ZigguratTables | None = None, source: UniformSource | None = None,
                 exp_tables: ZigguratTables | None = None, device=None):
        if tables is None:
            tables = default_tables(HALF_NORMAL)
        if tables.distribution != HALF_NORMAL:
            raise ValueError(f"need half-normal tables, got {tables.distribution!r}")
        if exp_tables is None:
            exp_tables = default_tables(EXPONENTIAL)
        super().__init__(tables, exp_tables, source, device)

    @property
    def tail_start(self) -> float:
        return float(self.tables.x[1])

    def overhang_attempt(self, j: int, ux: float, uy: float):
        """One plain-rejection box attempt (host probe)."""
        if not 1 <= j <= self.tables.l_max:
            raise IndexError(f"bounded slot out of range: {j}")
        xl, xr, fb, ft = self.tables.box_bounds(j)
        x = xl + ux * (xr - xl)
        if fb + uy * (ft - fb) < np.exp(-0.5 * x * x):
            return True, x, True
        return False, None, True
