"""Seeded 64-bit uniform sources (mirror of `zigfast/uniform.py`).

Generators, selected by the reference's integer ids (`uniform.py:22-26`):

* ``"xoshiro256++"`` (gid 0, the reference default) -- sequential stream; on
  the device it is produced in parallel blocks via GF(2) jump-ahead.
* ``"splitmix64"`` (gid 1) -- sequential stream, random-access by nature.
* replay (gid 2) -- a fixed word list played back with wrap-around.
* ``"ctr"`` (gid 3, new) -- the production counter stream: sample K of a fill
  reads word K = fmix64(seed + (K+1)*gamma) (MurmurHash3's finalizer on
  splitmix64's Weyl sequence), and its rare extra words come from the
  disjoint positions 2^63 + K*2^19 + t.  Output K depends only on (seed, K),
  never on launch shape or GPU count; the state is ``[seed, next_counter]``.

Host-side bookkeeping (seeding, cursors) is plain Python like the reference's;
word generation (`next_block`) runs on the GPU through the C-ABI.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import _lib
from .errors import BitBudgetExceeded

_MASK64 = (1 << 64) - 1

GENERATOR_IDS = {
    "xoshiro256++": _lib.GEN_XOSHIRO,
    "splitmix64": _lib.GEN_SPLITMIX,
    "replay": _lib.GEN_REPLAY,
    "ctr": _lib.GEN_CTR,
}

SEED_ENV_VAR = "ZIGFAST_SEED"
MAX_REUSED_BITS = 12
CTR_LIMIT = 1 << 44  # primary counter range of the "ctr" generator


def _splitmix64(state: int) -> tuple[int, int]:
    state = (state + 0x9E3779B97F4A7C15) & _MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return state, z ^ (z >> 31)


def _mix(h: int, v: int) -> int:
    return _splitmix64((h ^ (v & _MASK64)) & _MASK64)[1]


def auto_seed_value() -> int:
    """``ZIGFAST_SEED`` if set, else a hash of time and PIDs (`uniform.py:48-60`)."""
    env = os.environ.get(SEED_ENV_VAR)
    if env is not None:
        return int(env) & _MASK64
    try:
        ppid = os.getppid()
    except OSError:
        ppid = 0x5DEECE66D
    h = _mix(0, time.time_ns())
    h = _mix(h, os.getpid())
    return _mix(h, ppid)


def split_index(u: int, bits: int) -> tuple[int, int]:
    """Low ``bits`` of ``u`` plus the unmodified word (`uniform.py:63-73`)."""
    if bits < 1:
        raise ValueError("bits must be >= 1")
    if bits > MAX_REUSED_BITS:
        raise BitBudgetExceeded(f"cannot reuse {bits} low bits; limit is {MAX_REUSED_BITS}")
    return u & ((1 << bits) - 1), u


def derive_seed(base: int, stream: int) -> int:
    """Decorrelated per-shard seed (`uniform.py:132-134`)."""
    return _mix(_mix(0, base), 0x5851F42D4C957F2D + stream)


def xoshiro_seed_state(seed: int) -> np.ndarray:
    s, words = seed & _MASK64, []
    for _ in range(4):
        s, w = _splitmix64(s)
        words.append(w)
    return np.array(words, dtype=np.uint64)


class UniformSource:
    """Single-owner 64-bit word stream; not thread-safe (`uniform.py:76-81`)."""

    def __init__(self, seed: int | None = None, generator: str = "xoshiro256++"):
        if generator not in GENERATOR_IDS:
            raise ValueError(f"unknown generator: {generator!r}")
        if generator == "replay":
            raise ValueError("use UniformSource.replay() for replay sources")
        self.generator_id = generator
        self.gid = GENERATOR_IDS[generator]
        if seed is None:
            seed = auto_seed_value()
        self.seed = int(seed) & _MASK64
        if generator == "xoshiro256++":
            self.state = xoshiro_seed_state(self.seed)
        elif generator == "splitmix64":
            self.state = np.array([self.seed], dtype=np.uint64)
        else:
            self.state = np.array([self.seed, 0], dtype=np.uint64)
        self._words_dev = None

    @classmethod
    def replay(cls, words) -> "UniformSource":
        """Play back ``words`` verbatim, wrapping (`uniform.py:102-113`)."""
        src = object.__new__(cls)
        src.generator_id = "replay"
        src.gid = GENERATOR_IDS["replay"]
        src.seed = 0
        arr = np.asarray(words, dtype=np.uint64)
        if arr.size == 0:
            raise ValueError("replay source needs at least one word")
        src.state = np.concatenate([np.zeros(1, dtype=np.uint64), arr])
        src._words_dev = None
        return src

    @classmethod
    def counter(cls, seed: int | None = None, counter: int = 0) -> "UniformSource":
        """A production ("ctr") source positioned at sample ``counter``."""
        src = cls(seed, generator="ctr")
        src.state[1] = np.uint64(counter)
        return src

    # -- device plumbing -------------------------------------------------------
    def replay_words_device(self, device):
        """The replay word list as a device tensor (uploaded once per device)."""
        import torch
        if self._words_dev is None or self._words_dev.device != torch.device(device):
            host = torch.from_numpy(self.state[1:].view(np.int64).copy())
            self._words_dev = host.to(device)
        return self._words_dev

    def next_block_device(self, n: int, device=None):
        """``n`` words as an int64-viewed CUDA tensor, advancing the stream."""
        import torch
        device = torch.device(device if device is not None else "cuda")
        if self.gid == _lib.GEN_REPLAY:
            host = torch.from_numpy(self.next_block(n).view(np.int64))
            return host.to(device)
        out = torch.empty(n, dtype=torch.int64, device=device)
        with torch.cuda.device(device):
            _lib.check(_lib.lib().zf_words(self.gid, _lib.u64p(self.state), n, out.data_ptr(),
                                           _lib.stream_handle(device)))
        return out

    # -- reference API -----------------------------------------------------------
    def next_u64(self) -> int:
        return int(self.next_block(1)[0])

    def next_block(self, n: int) -> np.ndarray:
        if self.gid == _lib.GEN_REPLAY:
            words = self.state[1:]
            pos = int(self.state[0])
            idx = (pos + np.arange(n, dtype=np.uint64)) % np.uint64(words.size)
            self.state[0] = np.uint64(pos + n)
            return words[idx.astype(np.int64)]
        if n == 0:
            return np.empty(0, dtype=np.uint64)
        return self.next_block_device(n).cpu().numpy().view(np.uint64)

    def clone(self) -> "UniformSource":
        src = object.__new__(UniformSource)
        src.generator_id = self.generator_id
        src.gid = self.gid
        src.seed = self.seed
        src.state = self.state.copy()
        src._words_dev = self._words_dev
        return src

    def jump(self, k: int) -> None:
        """Skip ``k`` words ahead in O(log k) (xoshiro via GF(2) jump polynomials)."""
        if self.gid == _lib.GEN_XOSHIRO:
            _lib.check(_lib.lib().zf_xoshiro_jump(_lib.u64p(self.state), k))
        elif self.gid == _lib.GEN_SPLITMIX:
            self.state[0] = np.uint64((int(self.state[0]) + k * 0x9E3779B97F4A7C15) & _MASK64)
        elif self.gid == _lib.GEN_REPLAY:
            self.state[0] = np.uint64(int(self.state[0]) + k)
        else:
            self.state[1] = np.uint64(int(self.state[1]) + k)
