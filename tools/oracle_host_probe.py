"""Where an oracle-mode fill's time goes (experiment tool): the C-ABI call
alone (zf_fill_gid, xoshiro256++, preallocated output) vs the Python
sampler path, n = 1e6."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1403_6870_b200 as zf
from paper_1403_6870_b200 import _lib

dev = torch.device("cuda", 0)
n = 1_000_000
out = torch.empty(n, dtype=torch.float64, device=dev)
L = _lib.lib()
tabs = _lib.device_tables(zf.default_tables("exponential"), zf.default_tables("halfnormal"), 0)
st = zf.UniformSource(42).state.copy()
for label, fn in (
    ("C-ABI zf_fill_gid", lambda: L.zf_fill_gid(tabs.handle, 0, 0, 0, _lib.u64p(st), None, 0,
                                                  out.data_ptr(), n, None, None, None)),
    ("sampler.fill", lambda: zf.ExpSampler(source=zf.UniformSource(42), device=dev).fill(out)),
    ("zf_words 1.06M", lambda: L.zf_words(0, _lib.u64p(st), 1_060_000, out.data_ptr(), None)),
):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label:22s} median {np.median(ts) * 1e6:7.1f} us  min {min(ts) * 1e6:7.1f} us", flush=True)
