"""Generator-level statistical battery of the production word function (GPU).

    python tools/battery.py [--log2n 36] [--fns 0,1] [--seeds 7,1234] [--out file.json]

Runs the tests of tools/battery.cu on the counter stream words
w_K = f(seed + (K + 1) * gamma) for f = mix13 (FN 0, splitmix64's output
function, the round-1 production words) and f = fmix64 (FN 1, MurmurHash3's
finalizer, the round-2 production words) side by side, and reports chi-square
statistics with p-values (scipy).  The lags cover the kernel's sample layout:
1 and 2 (neighbours), 16 (one lane's samples), 64 (one warp iteration), 512
(one tile), 4096 and 2^19 (the secondary-stream spacing of one sample).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import pathlib
import subprocess
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
SO = HERE / "_build" / "libbattery.so"
KINDS = {0: "monobit", 1: "top6-pair", 2: "byte-pair", 3: "byte-vs-top6", 4: "hw-triple",
         5: "nibble-triple", 6: "top12-uniform", 7: "gap-0xFF"}
LAGS = (1, 2, 16, 64, 512, 4096, 1 << 19)


def build():
    SO.parent.mkdir(exist_ok=True)
    src = HERE / "battery.cu"
    if SO.exists() and SO.stat().st_mtime >= src.stat().st_mtime:
        return SO
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                    "-Xcompiler", "-fPIC", "-o", str(SO), str(src)], check=True)
    return SO


def chi2_p(stat, df):
    from scipy.stats import chi2
    return float(chi2.sf(stat, df))


def pooled_chi2(obs, exp):
    """Pearson chi-square with cells of expectation < 5 pooled left to right."""
    po, pe, ao, ae = [], [], 0.0, 0.0
    for o, e in zip(obs, exp):
        ao += o
        ae += e
        if ae >= 5.0:
            po.append(ao)
            pe.append(ae)
            ao = ae = 0.0
    if ae > 0 and pe:
        po[-1] += ao
        pe[-1] += ae
    po, pe = np.array(po), np.array(pe)
    return float(((po - pe) ** 2 / pe).sum()), len(pe) - 1


def expected(kind, n, total):
    if kind in (1, 2, 3, 5, 6):
        return np.full(4096, total / 4096.0)
    if kind == 4:
        from scipy.stats import binom
        pk = [binom.cdf(28, 64, .5), binom.cdf(31, 64, .5) - binom.cdf(28, 64, .5),
              binom.pmf(32, 64, .5), binom.cdf(35, 64, .5) - binom.cdf(32, 64, .5),
              binom.sf(35, 64, .5)]
        e = np.array([pk[a] * pk[b] * pk[c] for a in range(5) for b in range(5) for c in range(5)])
        return np.concatenate([e * total, np.zeros(4096 - 125)])
    if kind == 7:
        p = 1.0 / 256.0
        g = np.arange(4096, dtype=np.float64)
        e = p * (1 - p) ** g
        e[4095] = (1 - p) ** 4095
        return e * total
    raise ValueError(kind)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=36)
    ap.add_argument("--fns", default="0,1")
    ap.add_argument("--seeds", default="7,1234")
    ap.add_argument("--aval-log2m", type=int, default=22)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    L = C.CDLL(str(build()))
    L.bat_avalanche.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int]
    L.bat_stream.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                             C.c_void_p, C.c_int]
    cnt = torch.zeros(4096, dtype=torch.int64, device="cuda")
    n = 1 << a.log2n
    grid = max(148 * 8, n >> 24)
    rows = []
    for fn in (int(x) for x in a.fns.split(",")):
        name = "mix13" if fn == 0 else "fmix64"
        # avalanche of the word function on Weyl inputs
        m = 1 << a.aval_log2m
        cnt.zero_()
        assert L.bat_avalanche(fn, 7, m, cnt.data_ptr(), 148 * 8) == 0
        c = cnt.cpu().numpy().astype(np.float64)
        bias = c / m - 0.5
        stat = float(((c - m / 2) ** 2 / (m / 4)).sum())
        rows.append({"fn": name, "test": "avalanche", "m": m, "max_abs_bias": float(np.abs(bias).max()),
                     "rms_bias": float(np.sqrt((bias ** 2).mean())), "chi2": stat, "df": 4096,
                     "p": chi2_p(stat, 4096)})
        print(json.dumps(rows[-1]), flush=True)
        for seed in (int(x) for x in a.seeds.split(",")):
            plan = [(0, 0), (3, 0), (6, 0), (7, 0)] + [(k, lag) for k in (1, 2, 4, 5) for lag in LAGS]
            for kind, lag in plan:
                cnt.zero_()
                t0 = time.perf_counter()
                assert L.bat_stream(fn, kind, seed, 0, n, lag, cnt.data_ptr(), grid) == 0
                c = cnt.cpu().numpy().astype(np.float64)
                dt = time.perf_counter() - t0
                if kind == 0:
                    stat = float(((c[:64] - n / 2) ** 2 / (n / 4)).sum())
                    df = 64
                    worst = float(np.abs((c[:64] - n / 2) / math.sqrt(n / 4)).max())
                    extra = {"max_abs_z": worst}
                else:
                    total = c.sum()
                    e = expected(kind, n, total)
                    keep = e > 0
                    stat, df = pooled_chi2(c[keep], e[keep])
                    extra = {"events": int(total)}
                r = {"fn": name, "test": KINDS[kind], "seed": seed, "lag": lag, "n": n,
                     "chi2": stat, "df": df, "z": (stat - df) / math.sqrt(2 * df),
                     "p": chi2_p(stat, df), "seconds": round(dt, 2), **extra}
                rows.append(r)
                print(json.dumps(r), flush=True)
    if a.out:
        pathlib.Path(a.out).write_text(json.dumps(rows, indent=1))
    for name in ("mix13", "fmix64"):
        ps = [r["p"] for r in rows if r["fn"] == name and r["test"] != "avalanche"]
        if ps:
            print(f"{name}: {len(ps)} stream tests, min p {min(ps):.3g}, "
                  f"p<1e-3: {sum(p < 1e-3 for p in ps)}, p>1-1e-3: {sum(p > 1 - 1e-3 for p in ps)}")


if __name__ == "__main__":
    sys.exit(main())
