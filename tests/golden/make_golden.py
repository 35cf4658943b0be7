"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/golden.json.  Nothing at test time reads /root/reference;
the GPU box only sees this committed file.  Contents (all floats as IEEE-754
bit patterns in hex, so comparisons are bit-exact):

* the reference's own golden vectors (tests/test_uniform.py:14-23,
  tests/test_exp_sampler.py:10-16, tests/test_normal_sampler.py:10-16) and its
  replay known-answer cases (test_exp_sampler.py:93-108,
  test_normal_sampler.py:54-65), re-derived by calling the reference;
* alias arrays built by the reference (`alias.py:32-63`) for both tables;
* config 1 (BASELINE.json): Exponential, n = 1e6, UniformSource(42): SHA-256
  digests of the values and of the per-sample path records (start offset,
  words, layer byte, path bits, box attempts), counters, words consumed, plus
  head/tail samples; the same for the normal sampler on the same stream;
* production ("ctr") stream samples evaluated BY THE REFERENCE through replay
  of each sample's word sequence [S(K), S(2^63 + K*2^19 + t) ...],
  S(c) = fmix64(seed + (c+1) * gamma);
* derive_seed values and aggregate() sums;
* the traditional baseline (traditional.py, _kernels.py:933-1277): solved
  tables and packs, golden draws (tests/test_traditional.py:15-29), fills,
  counters, replay KATs, a config-1-sized record digest and production-stream
  samples evaluated through replay;
* run_quality moments (quality.py:109-138) for one shard and derive_seed
  shards.

It also exports the reference's solved traditional tables and packs to
paper_1403_6870_b200/data/traditional_256.npz (the product loads them).
"""
import hashlib
import json
import pathlib
import sys

import numpy as np

from zigfast import (ExpSampler, NormalSampler, TraditionalExpSampler, TraditionalNormalSampler,
                     UniformSource, derive_seed, run_quality, solve_traditional)
from zigfast.densities import exponential, half_normal
from zigfast.traditional import _pack as trad_pack
from zigfast._packs import make_alias
from zigfast.tables import default_tables

OUT = pathlib.Path(__file__).resolve().parent / "golden.json"
M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def hexbits(a) -> list:
    return [format(int(x), "016x") for x in np.asarray(a, dtype=np.float64).view(np.uint64)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fmix64(z):
    z = ((z ^ (z >> 33)) * 0xff51afd7ed558ccd) & M64
    z = ((z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53) & M64
    return z ^ (z >> 33)


def ctr_word(seed, c):
    """Production counter-stream word c: MurmurHash3's fmix64 on splitmix64's
    Weyl sequence (zf_device.cuh: fmix64)."""
    return fmix64((seed + (c + 1) * GAMMA) & M64)


def ctr_words(seed, K, m):
    base = (1 << 63) + (K << 19)
    return [ctr_word(seed, K)] + [ctr_word(seed, base + t) for t in range(m - 1)]


def records(cls, words, n):
    """Per-sample path records from the reference: replay cursor + counter deltas."""
    s = cls(source=UniformSource.replay(words))
    starts = np.empty(n, np.uint64)
    nw = np.empty(n, np.uint32)
    layer = np.empty(n, np.uint8)
    path = np.empty(n, np.uint8)
    att = np.empty(n, np.uint16)
    vals = np.empty(n)
    is_normal = cls is NormalSampler
    for k in range(n):
        p0 = int(s.source.state[0])
        c0 = s.counters.copy()
        vals[k] = s.sample_counted()
        d = s.counters - c0
        starts[k] = p0
        nw[k] = int(s.source.state[0]) - p0
        layer[k] = int(words[p0 % len(words)]) & 0xFF
        bits = 0
        if d[4]:
            bits |= 2                       # tail
        if d[1]:
            bits |= 1                       # exit through the common path
        elif d[2]:
            bits |= 4                       # overhang fast accept (exp)
        elif not (is_normal and d[4]):
            bits |= 8                       # accepted after a density evaluation
        path[k] = bits
        att[k] = d[5]
    return vals, starts, nw, layer, path, att, s.counters.copy(), int(s.source.state[0])


def trad_records(cls, words, n):
    """Per-sample records of the traditional samplers (slots 0 draws, 1 fast,
    2 wedge tests, 3 tails): exit path = tail / fast / wedge accept."""
    s = cls(source=UniformSource.replay(words))
    starts = np.empty(n, np.uint64)
    nw = np.empty(n, np.uint32)
    layer = np.empty(n, np.uint8)
    path = np.empty(n, np.uint8)
    att = np.empty(n, np.uint16)
    vals = np.empty(n)
    for k in range(n):
        p0 = int(s.source.state[0])
        c0 = s.counters.copy()
        vals[k] = s.sample_counted()
        d = s.counters - c0
        starts[k] = p0
        nw[k] = int(s.source.state[0]) - p0
        layer[k] = int(words[p0 % len(words)]) & 0xFF
        path[k] = 2 if d[3] else (1 if d[1] else 8)
        att[k] = d[2]
    return vals, starts, nw, layer, path, att, s.counters.copy(), int(s.source.state[0])


def traditional(g, words):
    for kind, fn, name, cls in (("exponential", exponential, "trad_exp", TraditionalExpSampler),
                                ("halfnormal", half_normal, "trad_normal",
                                 TraditionalNormalSampler)):
        t = solve_traditional(fn(), 256)
        se, kk, flo, fh, r = trad_pack(t, signed=(kind == "halfnormal"))
        g[f"{name}_tables"] = {
            "r": hexbits([t.r])[0], "v": hexbits([t.v])[0], "x_sha256": sha(t.x),
            "f_sha256": sha(t.f), "k_sha256": sha(t.k), "se_sha256": sha(se),
            "kk_sha256": sha(kk.astype(np.uint64)), "flo_sha256": sha(flo), "fh_sha256": sha(fh),
            "kk0": int(kk[0]), "fast_accept_probability": t.fast_accept_probability()}
        s = cls(source=UniformSource(7))
        g[f"{name}_seed7_first5"] = hexbits([s.sample() for _ in range(5)])
        g[f"{name}_seed7_fill3000"] = hexbits(cls(source=UniformSource(7)).fill(3000))
        g[f"{name}_splitmix99_fill2000"] = hexbits(
            cls(source=UniformSource(99, generator="splitmix64")).fill(2000))
        c = cls(source=UniformSource(3))
        c.fill_counted(200_000)
        g[f"{name}_seed3_counts200k"] = [int(x) for x in c.counters]
        g[f"{name}_seed11_aggregate20000"] = hexbits(
            [cls(source=UniformSource(11)).aggregate(20000)])[0]
        # replay KATs: fast accept, tail, wedge reject + restart
        kat = {}
        for label, w in (("fast", [123456789 << 8]),
                         ("tail", [0xFFFFFFFFFFFFFF00, 0x0123456789ABCDEF]),
                         ("tail_neg", [0x8000000000000100 - 0x100, 0x0123456789ABCDEF,
                                       0xFEDCBA9876543210] * 4),
                         ("wedge", [0xFFFFFFFFFFFFFF05, 0xFFFFFFFFFFFFFFFF, 42 << 8])):
            rs = cls(source=UniformSource.replay(w))
            kat[label] = {"words": [format(x, "016x") for x in w],
                          "value": hexbits([rs.sample()])[0], "cursor": int(rs.source.state[0])}
        g[f"{name}_kat"] = kat
        n1 = 1_000_000
        vals, starts, nw, layer, path, att, cnt, used = trad_records(cls, words, n1)
        ref = cls(source=UniformSource(42)).fill(n1)
        assert np.array_equal(ref.view(np.uint64), vals.view(np.uint64))
        g[f"c1_{name}"] = {
            "n": n1, "values_sha256": sha(vals), "starts_sha256": sha(starts),
            "nwords_sha256": sha(nw), "layer_sha256": sha(layer), "path_sha256": sha(path),
            "attempts_sha256": sha(att) if name == "trad_exp" else None,
            "counters": [int(x) for x in cnt], "words_consumed": used,
            "head": hexbits(vals[:64]), "tail": hexbits(vals[-64:]),
            "tail_positions": [int(i) for i in np.nonzero(path == 2)[0][:2000]],
            "n_exceptional": int((nw > 1).sum()),
        }
        print(name, "config-1 digests done", cnt, used, file=sys.stderr)
        out = {}
        for seed, base, count in ((1234, 0, 4096), (7, 1 << 40, 2048)):
            vv = []
            for k in range(count):
                w = ctr_words(seed, base + k, 64)
                rs = cls(source=UniformSource.replay(w))
                vv.append(rs.sample())
                assert int(rs.source.state[0]) <= len(w)
            out[f"{seed}:{base}"] = hexbits(vv)
        g[f"ctr_{name}"] = out


def export_traditional():
    """The solved traditional tables and packs (traditional.py:56-121) as a
    package fixture, so the product loads them instead of re-solving."""
    arrays = {}
    for kind, fn in (("exponential", exponential), ("halfnormal", half_normal)):
        t = solve_traditional(fn(), 256)
        se, kk, flo, fh, r = trad_pack(t, signed=(kind == "halfnormal"))
        arrays.update({f"{kind}_x": t.x, f"{kind}_f": t.f, f"{kind}_k": t.k,
                       f"{kind}_rv": np.array([t.r, t.v]), f"{kind}_se": se,
                       f"{kind}_kk": np.asarray(kk, dtype=np.uint64), f"{kind}_flo": flo,
                       f"{kind}_fh": fh})
    out = OUT.parent.parent.parent / "paper_1403_6870_b200" / "data" / "traditional_256.npz"
    np.savez(out, **arrays)
    print("wrote", out, file=sys.stderr)


def main():
    g = {}
    g["xoshiro_12345_first8"] = [int(w) for w in UniformSource(12345).next_block(8)]
    g["xoshiro_42_first64"] = [format(int(w), "016x") for w in UniformSource(42).next_block(64)]
    g["splitmix_42_first32"] = [format(int(w), "016x")
                                for w in UniformSource(42, generator="splitmix64").next_block(32)]
    words = UniformSource(42).next_block(1_100_000)
    g["xoshiro_42_1p1M_sha256"] = sha(words)
    src = UniformSource(42)
    src.next_block(1_000_000)
    g["xoshiro_42_after_1M_state"] = [format(int(w), "016x") for w in src.state]

    for kind in ("exponential", "halfnormal"):
        a = make_alias(default_tables(kind))
        g[f"alias_{kind}_prob"] = hexbits(a.prob)
        g[f"alias_{kind}_alias"] = [int(x) for x in a.alias]

    for name, cls in (("exp", ExpSampler), ("normal", NormalSampler)):
        s = cls(source=UniformSource(7))
        g[f"{name}_seed7_first5"] = hexbits([s.sample() for _ in range(5)])
        g[f"{name}_seed7_fill3000"] = hexbits(cls(source=UniformSource(7)).fill(3000))
        g[f"{name}_splitmix99_fill2000"] = hexbits(
            cls(source=UniformSource(99, generator="splitmix64")).fill(2000))
        c = cls(source=UniformSource(3))
        c.fill_counted(200_000)
        g[f"{name}_seed3_counts200k"] = [int(x) for x in c.counters]
        g[f"{name}_seed11_aggregate20000"] = format(
            int(np.float64(cls(source=UniformSource(11)).aggregate(20000)).view(np.uint64)), "016x")

    # replay KATs
    word = 123456789 << 8
    e = default_tables("exponential")
    g["kat_exp_common"] = hexbits([ExpSampler(source=UniformSource.replay([word])).sample()])
    g["kat_exp_tail"] = hexbits([ExpSampler(source=UniformSource.replay([255, 0, 0, word])).sample()])
    g["kat_normal_common"] = hexbits([NormalSampler(source=UniformSource.replay([word])).sample()])
    g["kat_normal_neg"] = hexbits(
        [NormalSampler(source=UniformSource.replay([(1 << 63) | word])).sample()])
    g["kat_word"] = word
    g["exp_x1"] = hexbits([e.x[1]])
    # wrap-around replay: 7 words, 40 draws (exercises modulo + exceptional)
    wrapw = [0xFF, 0x12345600, 0x0, 0xFE, 0xABCDEF01, 0x7F00, 0xFFFFFFFFFFFFFFFF]
    for name, cls in (("exp", ExpSampler), ("normal", NormalSampler)):
        s = cls(source=UniformSource.replay(wrapw))
        g[f"{name}_wrap_fill40"] = hexbits(s.fill(40))
        g[f"{name}_wrap_cursor"] = int(s.source.state[0])
    g["wrap_words"] = [format(w, "016x") for w in wrapw]

    # config 1 and its normal twin: digests of values and per-sample records
    n1 = 1_000_000
    for name, cls in (("exp", ExpSampler), ("normal", NormalSampler)):
        vals, starts, nw, layer, path, att, cnt, used = records(cls, words, n1)
        ref = cls(source=UniformSource(42)).fill(n1)
        assert np.array_equal(ref.view(np.uint64), vals.view(np.uint64))
        g[f"c1_{name}"] = {
            "n": n1, "values_sha256": sha(vals), "starts_sha256": sha(starts),
            "nwords_sha256": sha(nw), "layer_sha256": sha(layer), "path_sha256": sha(path),
            "attempts_sha256": sha(att) if name == "exp" else None,
            # the normal counted kernel counts box attempts only (slot 5,
            # _kernels.py:681), so tail samples record 0 there
            "attempts_box_sha256": sha(np.where(path & 2, 0, att).astype(np.uint16)),
            "counters": [int(x) for x in cnt], "words_consumed": used,
            "head": hexbits(vals[:64]), "tail": hexbits(vals[-64:]),
            "n_exceptional": int((nw > 1).sum()),
        }
        print(name, "config-1 digests done", cnt, used, file=sys.stderr)

    # production counter stream, evaluated by the reference through replay
    for name, cls in (("exp", ExpSampler), ("normal", NormalSampler)):
        out = {}
        for seed, base, count in ((1234, 0, 4096), (7, 1 << 40, 2048), (99, (1 << 44) - 4096, 4096)):
            vals = []
            for k in range(count):
                w = ctr_words(seed, base + k, 96)
                s = cls(source=UniformSource.replay(w))
                vals.append(s.sample())
                assert int(s.source.state[0]) <= len(w)
            out[f"{seed}:{base}"] = hexbits(vals)
        g[f"ctr_{name}"] = out

    traditional(g, words)
    export_traditional()

    # run_quality (quality.py:109-138): moments of the reference's own streams,
    # one shard and derive_seed shards
    rq = {}
    for dist in ("normal", "exp"):
        for jobs, n, chunk in ((4, 1 << 20, 1 << 22), (1, 1 << 20, 1 << 18), (3, 100_003, 4096)):
            r = run_quality(dist, n, seed=7, jobs=jobs, chunk=chunk)
            rq[f"{dist}:{n}:{jobs}:{chunk}"] = {"moments": hexbits(r.moments),
                                                "passed": bool(r.passed)}
    g["run_quality_seed7"] = rq
    g["derive_seed"] = {f"{b}:{s}": derive_seed(b, s) for b in (0, 123, 1234, M64) for s in (0, 1, 7)}
    OUT.write_text(json.dumps(g, indent=0))
    print("wrote", OUT, OUT.stat().st_size, "bytes", file=sys.stderr)


if __name__ == "__main__":
    main()
