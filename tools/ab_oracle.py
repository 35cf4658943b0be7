"""A/B of library builds on oracle-mode fills (experiment tool, not product).

    python tools/ab_oracle.py [--n 26] [--rounds 5] [--reps 5] lib_a.so lib_b.so ...

xoshiro256++ seed 42 through zf_fill_gid (gid 0), exp and normal; wall time
per fill (the call synchronises); outputs compared with the first library's.
"""
import argparse
import ctypes as C
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=26)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    from paper_1403_6870_b200.uniform import xoshiro_seed_state
    n = 1 << a.n
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    runs, ref = [], {}
    u64p = C.POINTER(C.c_uint64)
    for p in a.libs:
        L = C.CDLL(p)
        L.zf_tables_create_default.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.zf_fill_gid.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, u64p, C.c_void_p,
                                  C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                  C.c_void_p]
        h = C.c_void_p()
        assert L.zf_tables_create_default(0, C.byref(h)) == 0
        for d in (0, 1):
            st = xoshiro_seed_state(42)
            assert L.zf_fill_gid(h, d, 0, 0, st.ctypes.data_as(u64p), None, 0, out.data_ptr(), n,
                                 None, None, None) == 0
            torch.cuda.synchronize()
            sig = (out[:1000].cpu().numpy().tobytes(), st.tobytes())
            if d not in ref:
                ref[d] = sig
            elif sig != ref[d]:
                print(f"!! {p} differs (dist {d})", flush=True)
        runs.append((p, L, h, {0: [], 1: []}))
    for _ in range(a.rounds):
        for p, L, h, ts in runs:
            for d in (0, 1):
                st = xoshiro_seed_state(42)
                time.sleep(0.05)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(a.reps):
                    L.zf_fill_gid(h, d, 0, 0, st.ctypes.data_as(u64p), None, 0, out.data_ptr(), n,
                                  None, None, None)
                torch.cuda.synchronize()
                ts[d].append((time.perf_counter() - t0) / a.reps)
    for p, _, _, ts in runs:
        for d, name in ((0, "exp"), (1, "normal")):
            m = statistics.median(ts[d])
            print(f"{p.split('/')[-1]:16s} {name:6s} n=2^{a.n}: {m * 1e3:.3f} ms  {n / m / 1e9:.1f} G/s",
                  flush=True)


if __name__ == "__main__":
    main()
