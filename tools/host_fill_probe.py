"""Throughput of fill(numpy array) -- pageable host destinations through the
pinned staging path -- for a few staging chunk sizes."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
import paper_1403_6870_b200 as zf
from paper_1403_6870_b200 import samplers

n = 1 << 26
for mb in [int(x) for x in os.environ.get("STAGE_MB", "64").split(",")]:
    samplers._STAGE_BYTES = mb << 20
    samplers._stage_cache.clear()
    for gen in ("ctr", "xoshiro256++"):
        for dt in (np.float64, np.float32):
            a = np.empty(n, dtype=dt)
            src = zf.UniformSource.counter(1) if gen == "ctr" else zf.UniformSource(1)
            s = zf.NormalSampler(source=src)
            s.fill(a)
            t = time.perf_counter()
            for _ in range(3): s.fill(a)
            dt_ = (time.perf_counter() - t) / 3
            print(f"stage {mb} MB {gen} {a.dtype} numpy fill 2^26: {dt_*1e3:.1f} ms {n/dt_/1e9:.2f} G/s")
