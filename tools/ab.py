"""A/B several builds of the library in ONE process (experiment tool, not product).

    python tools/ab.py [--n 28] [--reps 20] [--rounds 5] [--dists normal,exp] \
                       [--dtype f64] lib_a.so lib_b.so ...

Every library is loaded with its own ctypes handle (RTLD_LOCAL), gets its own
default-table handle, and fills the same device buffer through `zf_fill` on
the legacy default stream.  Rounds interleave the libraries so clock drift
hits all of them alike; the median over rounds is reported.  Before timing,
each library's output on a 2^24-sample fill is compared bit for bit with the
first library's (a variant that changes values is flagged, not timed).
"""
from __future__ import annotations

import argparse
import ctypes as C
import statistics
import sys
import time

import torch


def load(path):
    L = C.CDLL(path)
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
    L.zf_tables_create_default.restype = i32
    L.zf_tables_create_default.argtypes = [i32, C.POINTER(vp)]
    L.zf_fill.restype = i32
    L.zf_fill.argtypes = [vp, i32, i32, u64, u64, vp, u64, vp, vp]
    h = vp()
    assert L.zf_tables_create_default(0, C.byref(h)) == 0
    return L, h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--dists", default="normal,exp")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the equal-output gate")
    ap.add_argument("--sustain", type=float, default=0.0,
                    help="instead of timed reps: run each lib/dist for this many seconds and "
                         "report the average rate and the energy per sample (NVML)")
    ap.add_argument("--cool", type=float, default=0.0,
                    help="idle seconds before each measurement (keeps the power average low)")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dt = torch.float64 if a.dtype == "f64" else torch.float32
    code = 0 if a.dtype == "f64" else 1
    n = 1 << a.n
    out = torch.empty(n, dtype=dt, device=dev)
    libs = [(p, *load(p)) for p in a.libs]
    dists = {"exp": 0, "normal": 1}
    # correctness gate: identical values on a small fill
    bad = set()
    for dname in a.dists.split(","):
        ref = None
        for p, L, h in libs:
            x = torch.empty(1 << 24, dtype=dt, device=dev)
            assert L.zf_fill(h, dists[dname], code, a.seed, 12345, x.data_ptr(), x.numel(),
                             None, None) == 0
            torch.cuda.synchronize()
            if ref is None:
                ref = x
            elif not torch.equal(x, ref) and not a.no_check:
                bad.add(p)
                print(f"!! {p} differs from {libs[0][0]} on {dname}", flush=True)
    if a.sustain:
        import pynvml as N
        N.nvmlInit()
        nvh = N.nvmlDeviceGetHandleByIndex(0)
        for r in range(a.rounds):
            for p, L, h in libs:
                for dname in a.dists.split(","):
                    d = dists[dname]
                    time.sleep(max(a.cool, 3.0))
                    torch.cuda.synchronize()
                    e0 = N.nvmlDeviceGetTotalEnergyConsumption(nvh)
                    t0 = time.perf_counter()
                    k = 0
                    while time.perf_counter() - t0 < a.sustain:
                        for _ in range(8):
                            L.zf_fill(h, d, code, a.seed, 0, out.data_ptr(), n, None, None)
                        k += 8
                        torch.cuda.synchronize()
                    dt = time.perf_counter() - t0
                    e1 = N.nvmlDeviceGetTotalEnergyConsumption(nvh)
                    clk = N.nvmlDeviceGetClockInfo(nvh, N.NVML_CLOCK_SM)
                    print(f"{p.split('/')[-1]:24s} {dname:6s} sustained {a.sustain:.1f}s: "
                          f"{k * n / dt / 1e9:7.1f} G/s, {(e1 - e0) * 1e-3 / dt:6.1f} W, "
                          f"{(e1 - e0) * 1e-3 / (k * n) * 1e9:.3f} nJ/sample, sm_mhz {clk}",
                          flush=True)
        return
    res = {(p, d): [] for p, _, _ in libs for d in a.dists.split(",")}
    clk = {(p, d): [] for p, _, _ in libs for d in a.dists.split(",")}
    try:
        import pynvml as N
        N.nvmlInit()
        nv = N.nvmlDeviceGetHandleByIndex(0)
        sm_clock = lambda: N.nvmlDeviceGetClockInfo(nv, N.NVML_CLOCK_SM)
    except Exception:
        sm_clock = lambda: 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(a.rounds):
        for p, L, h in libs:
            if p in bad:
                continue
            for dname in a.dists.split(","):
                d = dists[dname]
                if a.cool:
                    time.sleep(a.cool)
                for _ in range(2):
                    L.zf_fill(h, d, code, a.seed, 0, out.data_ptr(), n, None, None)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(a.reps):
                    L.zf_fill(h, d, code, a.seed, 0, out.data_ptr(), n, None, None)
                e1.record()
                c = sm_clock()
                torch.cuda.synchronize()
                res[(p, dname)].append(e0.elapsed_time(e1) / a.reps)
                clk[(p, dname)].append(c)
    for (p, dname), ms in res.items():
        if not ms:
            continue
        m = statistics.median(ms)
        cl = clk[(p, dname)]
        norm = statistics.median([x * c / 1965.0 for x, c in zip(ms, cl)]) if all(cl) else m
        print(f"{p.split('/')[-1]:24s} {dname:6s} @1965MHz-equivalent: {n / norm / 1e6:7.1f} G/s")
        print(f"{p.split('/')[-1]:24s} {dname:6s} n=2^{a.n} {a.dtype}: {m:.4f} ms  "
              f"{n / m / 1e6:7.1f} G/s (best {n / min(ms) / 1e6:7.1f}) sm_mhz "
              f"{statistics.median(clk[(p, dname)]):.0f} [{min(clk[(p, dname)])}-"
              f"{max(clk[(p, dname)])}]", flush=True)
        if a.verbose:
            print("   ", " ".join(f"{x:.4f}@{c}" for x, c in zip(ms, clk[(p, dname)])))


if __name__ == "__main__":
    sys.exit(main())
