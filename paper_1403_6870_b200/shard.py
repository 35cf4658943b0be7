"""Multi-GPU sharding of the production stream (BASELINE.json config 3).

Each rank owns a disjoint counter range of the same seed: rank r draws global
samples [r * 2^40 + c, ...), so the output of every rank depends only on
(seed, rank offset, counter) -- never on how many ranks run or how the grid is
shaped -- and no rank exchanges samples with another.  The only collective is
a SUM allreduce of the validation statistics (moment sums, histogram and
threshold counts), a few KB per run; nothing crosses NVLink on the hot path.
The reference's analogue is per-thread samplers seeded `derive_seed(base, i)`
merged with `math.fsum` (quality.py:121-129).
"""

from __future__ import annotations

import math

RANK_STRIDE = 1 << 40          # counter offset between ranks (config 3)
MAX_RANKS = 16                 # 16 * 2^40 = 2^44, the primary counter range


def counter_base(rank: int, start: int = 0) -> int:
    """First counter of ``rank``'s shard (``start`` = samples already drawn)."""
    if not 0 <= rank < MAX_RANKS:
        raise ValueError(f"rank {rank} outside the counter space (max {MAX_RANKS})")
    if not 0 <= start < RANK_STRIDE:
        raise ValueError("per-rank stream exhausted (2^40 samples)")
    return rank * RANK_STRIDE + start


def pack_stats(sums, hist, thresh_counts) -> list[float]:
    """Flatten statistics into one vector for a single allreduce.  Counts stay
    exact in float64 up to 2^53 (far above any per-run total here)."""
    return [float(s) for s in sums] + [float(h) for h in hist] + [float(c) for c in thresh_counts]


def unpack_stats(vec, nsums: int, nhist: int, nthresh: int):
    vec = list(vec)
    return (vec[:nsums], [int(round(v)) for v in vec[nsums:nsums + nhist]],
            [int(round(v)) for v in vec[nsums + nhist:nsums + nhist + nthresh]])


def allreduce_stats(vec, device=None, group=None):
    """SUM-allreduce a stats vector across the default process group (NCCL on
    GPUs, gloo on CPU); returns the reduced list.  No-op without a group."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vec, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().tolist()


def exact_sum(parts) -> float:
    return math.fsum(parts)
