"""Fixed per-call overhead of small fills through the Python API (experiment tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1403_6870_b200 as zf  # noqa: E402

dev = torch.device("cuda", 0)
out = torch.empty(1 << 20, dtype=torch.float64, device=dev)
for name, src in (("oracle", lambda: zf.UniformSource(42)), ("ctr", lambda: zf.UniformSource.counter(7))):
    s = zf.ExpSampler(source=src(), device=dev)
    for n in (1024, 1 << 20):
        o = out[:n]
        for _ in range(5):
            s.fill(o)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(50):
            s.fill(o)
        torch.cuda.synchronize()
        print(f"{name:6s} fill n={n:8d}: {(time.perf_counter() - t) / 50 * 1e6:7.1f} us per call")
    t = time.perf_counter()
    for _ in range(2000):
        s.sample()
    print(f"{name:6s} sample(): {(time.perf_counter() - t) / 2000 * 1e6:7.2f} us per call")
