"""Pinned D2H copy rate: one copy vs chunks spread over concurrent streams
(copy engines), for the e2e bound (experiment tool, not product).

    python tools/d2h_probe.py [log2 bytes]
"""
import sys
import time

import torch

nbytes = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 31)
n = nbytes // 8
dev = torch.device("cuda", 0)
host = torch.empty(n, dtype=torch.float64).pin_memory()
dbuf = torch.randn(n, dtype=torch.float64, device=dev)
streams = [torch.cuda.Stream(dev) for _ in range(8)]


def run(k, chunk_mb):
    chunk = chunk_mb * (1 << 20) // 8
    torch.cuda.synchronize()
    t = time.perf_counter()
    for r in range(3):
        i = 0
        j = 0
        while i < n:
            e = min(n, i + chunk)
            s = streams[j % k]
            with torch.cuda.stream(s):
                host[i:e].copy_(dbuf[i:e], non_blocking=True)
            i = e
            j += 1
    torch.cuda.synchronize()
    return 3 * nbytes / (time.perf_counter() - t) / 1e9


for k in (1, 2, 4):
    for c in (16, 64, 256, 2048):
        print(f"streams={k} chunk={c} MB: {run(k, c):.1f} GB/s", flush=True)
