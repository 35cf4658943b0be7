"""A/B of library builds on the config-4 batch (experiment tool, not product).

    python tools/ab_batch.py [--rounds 10] [--reps 20] lib_a.so lib_b.so ...

4096 requests x 8192 samples, alternating exp/normal, seeds 0..4095, resident
request table (zf_batch_create) per library; CUDA-event time per
zf_batch_fill; outputs compared with the first library's.
"""
import argparse
import ctypes as C
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1403_6870_b200 import _lib  # noqa: E402  (Request struct only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    m, per = 4096, 8192
    reqs = (_lib.Request * m)()
    for i in range(m):
        reqs[i] = _lib.Request(i, 0, per, i * per, i % 2, 0)
    out = torch.empty(m * per, dtype=torch.float64, device="cuda")
    ref = None
    runs = []
    for p in a.libs:
        L = C.CDLL(p)
        L.zf_tables_create_default.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.zf_batch_create.argtypes = [C.c_void_p, C.POINTER(_lib.Request), C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p)]
        L.zf_batch_fill.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        t, b = C.c_void_p(), C.c_void_p()
        assert L.zf_tables_create_default(0, C.byref(t)) == 0
        assert L.zf_batch_create(t, reqs, m, 0, C.byref(b)) == 0
        out.zero_()
        assert L.zf_batch_fill(b, C.c_void_p(out.data_ptr()), None) == 0
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        elif not torch.equal(out, ref):
            print(f"!! {p} differs", flush=True)
        runs.append((p, L, b, []))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(a.rounds):
        for p, L, b, ts in runs:
            time.sleep(0.05)
            for _ in range(3):
                L.zf_batch_fill(b, C.c_void_p(out.data_ptr()), None)
            e0.record()
            for _ in range(a.reps):
                L.zf_batch_fill(b, C.c_void_p(out.data_ptr()), None)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / a.reps)
    for p, _, _, ts in runs:
        print(f"{p.split('/')[-1]:16s} median {statistics.median(ts):7.2f} us  best {min(ts):7.2f} us"
              f"  ({m * per / statistics.median(ts) / 1e3:.1f} G samples/s)", flush=True)


if __name__ == "__main__":
    main()
