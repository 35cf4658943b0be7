"""Pin the CPU oracle to the reference: golden vectors from the reference's own
tests and fixtures produced by running the reference (tests/golden/make_golden.py)."""
import hashlib

import numpy as np
import pytest

from helpers import assert_bits_equal, bits, hex_to_bits


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# first eight xoshiro256++ outputs for seed 12345 (reference tests/test_uniform.py:14-23)
GOLDEN_12345 = [10201931350592234856, 3780764549115216544, 1570246627180645737,
                3237956550421933520, 4899705286669081817, 13385132719381623431,
                4322154809380817970, 14774873379570401602]
# reference tests/test_exp_sampler.py:10-16 and tests/test_normal_sampler.py:10-16
EXP_SEED7 = [0.15069938164952687, 0.70774302052625893, 1.3168329449999849,
             1.1723584574009387, 1.7174354047860962]
NORMAL_SEED7 = [0.22612838171099861, 0.88945758308515721, -0.91723712988337558,
                1.7531374769622967, -0.11601284545578643]


def test_xoshiro_golden_words(orc, golden):
    assert [int(w) for w in orc.words("xoshiro256++", 12345, 8)] == GOLDEN_12345
    assert golden["xoshiro_12345_first8"] == GOLDEN_12345
    assert [format(int(w), "016x") for w in orc.words("xoshiro256++", 42, 64)] == \
        golden["xoshiro_42_first64"]
    assert sha(orc.words("xoshiro256++", 42, 1_100_000)) == golden["xoshiro_42_1p1M_sha256"]


def test_splitmix_words(orc, golden):
    assert [format(int(w), "016x") for w in orc.words("splitmix64", 42, 32)] == \
        golden["splitmix_42_first32"]


def test_seed7_first_draws(orc):
    assert list(orc.fill_stream("exp", 5, seed=7)[0]) == EXP_SEED7
    assert list(orc.fill_stream("normal", 5, seed=7)[0]) == NORMAL_SEED7


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_fill_and_counts_match_reference(orc, golden, dist):
    assert_bits_equal(orc.fill_stream(dist, 3000, seed=7)[0],
                      hex_to_bits(golden[f"{dist}_seed7_fill3000"]), "seed 7")
    assert_bits_equal(orc.fill_stream(dist, 2000, generator="splitmix64", seed=99)[0],
                      hex_to_bits(golden[f"{dist}_splitmix99_fill2000"]), "splitmix 99")
    _, cnt, _, _ = orc.fill_stream(dist, 200_000, seed=3)
    assert cnt.tolist() == golden[f"{dist}_seed3_counts200k"]


def test_replay_known_answers(orc, golden):
    w = golden["kat_word"]
    assert_bits_equal(orc.fill_stream("exp", 1, replay_words=[w])[0],
                      hex_to_bits(golden["kat_exp_common"]))
    assert_bits_equal(orc.fill_stream("exp", 1, replay_words=[255, 0, 0, w])[0],
                      hex_to_bits(golden["kat_exp_tail"]))
    assert_bits_equal(orc.fill_stream("normal", 1, replay_words=[w])[0],
                      hex_to_bits(golden["kat_normal_common"]))
    assert_bits_equal(orc.fill_stream("normal", 1, replay_words=[(1 << 63) | w])[0],
                      hex_to_bits(golden["kat_normal_neg"]))


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_replay_wraps(orc, golden, dist):
    words = hex_to_bits(golden["wrap_words"])
    vals, _, _, used = orc.fill_stream(dist, 40, replay_words=words)
    assert_bits_equal(vals, hex_to_bits(golden[f"{dist}_wrap_fill40"]), "wrap")
    assert used == golden[f"{dist}_wrap_cursor"]


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_config1_values_and_paths(orc, golden, dist):
    """BASELINE config 1 (n = 1e6, UniformSource(42)): values AND per-sample
    path records identical to the reference's."""
    g = golden[f"c1_{dist}"]
    vals, cnt, recs, used = orc.fill_stream(dist, g["n"], seed=42, records=True)
    assert sha(vals) == g["values_sha256"]
    assert cnt.tolist() == g["counters"]
    assert used == g["words_consumed"]
    assert sha(recs["start"]) == g["starts_sha256"]
    assert sha(recs["nwords"]) == g["nwords_sha256"]
    assert sha(recs["layer"]) == g["layer_sha256"]
    assert sha(recs["path"]) == g["path_sha256"]
    if g["attempts_sha256"]:
        assert sha(recs["attempts"]) == g["attempts_sha256"]
    assert int((recs["nwords"] > 1).sum()) == g["n_exceptional"]


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_whole_output_checker_is_the_production_oracle(orc, golden, dist):
    """`check_ctr` (the multi-threaded in-place comparison the full-size GPU
    parity test uses) accepts the reference-evaluated production goldens and
    `fill_ctr`'s output in fp64 and fp32, and reports injected bit flips with
    the lowest index, whatever the thread split."""
    for key, want in golden[f"ctr_{dist}"].items():
        seed, base = (int(x) for x in key.split(":"))
        vals = hex_to_bits(want).view(np.float64)
        assert orc.check_ctr(dist, vals, seed, base) == (0, len(want)), key
    n = 300_007
    base = (1 << 40) + 11
    want, _, _ = orc.fill_ctr(dist, n, seed=7, ctr_base=base)
    for threads in (1, 3, 16):
        assert orc.check_ctr(dist, want, 7, base, threads=threads) == (0, n)
        assert orc.check_ctr(dist, want.astype(np.float32), 7, base, threads=threads) == (0, n)
    assert orc.check_ctr(dist, want, 8, base)[0] > n // 2  # another seed: nothing matches
    exc = np.flatnonzero(np.isin(np.arange(n), [5, 77_777, n - 1]))
    flipped = want.copy()
    flipped.view(np.uint64)[exc] ^= np.uint64(1)
    for threads in (1, 5):
        assert orc.check_ctr(dist, flipped, 7, base, threads=threads) == (3, 5)
    assert orc.check_ctr(dist, want[:0], 7, base) == (0, 0)


@pytest.mark.parametrize("dist,thr,use_abs", [("normal", (0.0, 1.0, 3.0, 3.7, 5.0), True),
                                              ("normal", (-1.0, 0.0, 2.5), False),
                                              ("exp", (0.5, 7.569274694148063, 9.0), False)])
def test_generate_and_count_is_the_production_oracle(orc, dist, thr, use_abs):
    """`count_ctr` (config 5's generate-and-count on the CPU, nothing stored)
    counts exactly what numpy counts on `fill_ctr`'s values, for any thread split."""
    n, base = 1_000_003, (5 << 40) + 9
    vals, _, _ = orc.fill_ctr(dist, n, seed=99, ctr_base=base)
    a = np.abs(vals) if use_abs else vals
    want = [int((a > t).sum()) for t in thr]
    for threads in (1, 7):
        assert orc.count_ctr(dist, n, 99, base, thr, use_abs, threads=threads) == want
    assert orc.count_ctr(dist, 0, 99, base, thr, use_abs) == [0] * len(thr)


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_production_stream_matches_reference_replay(orc, golden, dist):
    """The counter ("ctr") stream restated in C equals the reference run over
    each sample's word sequence."""
    for key, want in golden[f"ctr_{dist}"].items():
        seed, base = (int(x) for x in key.split(":"))
        vals, _, _ = orc.fill_ctr(dist, len(want), seed=seed, ctr_base=base)
        assert_bits_equal(vals, hex_to_bits(want), f"ctr {key}")


def test_alias_tables_match_reference(orc, golden):
    hn, ex = orc.packs()
    for kind, p in (("exponential", ex), ("halfnormal", hn)):
        assert_bits_equal(p.prob, hex_to_bits(golden[f"alias_{kind}_prob"]), kind)
        assert p.alias.tolist() == golden[f"alias_{kind}_alias"]


def test_derive_seed(orc, golden):
    for key, want in golden["derive_seed"].items():
        b, s = (int(x) for x in key.split(":"))
        assert orc.derive_seed(b, s) == want


def test_aggregate_is_sequential_sum(orc, golden):
    for dist in ("exp", "normal"):
        got = orc.aggregate(dist, 20000, 11)
        want = hex_to_bits([golden[f"{dist}_seed11_aggregate20000"]]).view(np.float64)[0]
        assert got == want
        vals = orc.fill_stream(dist, 20000, seed=11)[0]
        acc = 0.0
        for v in vals:
            acc += v
        assert acc == got


def test_sharded_baseline_is_reference_sharding(orc):
    """The CPU baseline's threads reproduce quality.py's derive_seed sharding."""
    n, threads = 10_000, 4
    out = orc.fill_sharded("exp", n, 5, threads=threads)
    off = 0
    for i in range(threads):
        share = n // threads + (1 if i < n % threads else 0)
        want = orc.fill_stream("exp", share, seed=orc.derive_seed(5, i))[0]
        assert np.array_equal(bits(out[off:off + share]), bits(want))
        off += share


@pytest.mark.parametrize("dist", ["exp", "normal"])
def test_sharded_fast_fill_equals_reference_fill(orc, dist):
    """The CPU baseline's register-resident fast fill (orc_fill_sharded) gives
    the same values as the general restatement, shard by shard
    (quality.py:121-126 sharding: shard i seeded derive_seed(seed, i))."""
    n, threads, seed = 300_001, 3, 1234
    got = orc.fill_sharded(dist, n, seed, threads=threads)
    off = 0
    for i in range(threads):
        share = n // threads + (1 if i < n % threads else 0)
        want, _, _, _ = orc.fill_stream(dist, share, seed=orc.derive_seed(seed, i))
        assert_bits_equal(got[off:off + share], bits(want), f"shard {i}")
        off += share


def _ref_run_quality_moments(orc, dist, n, seed, jobs, chunk):
    """quality.py:92-138 restated over the oracle's xoshiro256++ streams: jobs
    shards seeded derive_seed(seed, i), per-chunk numpy sums, fsum merge."""
    import math
    seeds = [seed] if jobs == 1 else [orc.derive_seed(seed, i) for i in range(jobs)]
    shares = [n] if jobs == 1 else [n // jobs + (1 if i < n % jobs else 0) for i in range(jobs)]
    sums = [[] for _ in range(5)]
    for sd, m in zip(seeds, shares):
        v = orc.fill_stream(dist, m, seed=sd)[0]
        for off in range(0, m, chunk):
            view = v[off:off + chunk]
            p = view
            for k in range(5):
                if k:
                    p = p * view
                sums[k].append(float(p.sum()))
    return [math.fsum(s) / n for s in sums]


def test_run_quality_golden_pinned_by_oracle(orc, golden):
    """The reference's run_quality moments (golden, produced by running it)
    equal the oracle restatement bit for bit: derive_seed sharding, share
    split, chunking and the fsum merge are pinned."""
    for key, want in golden["run_quality_seed7"].items():
        dist, n, jobs, chunk = key.split(":")
        got = _ref_run_quality_moments(orc, dist, int(n), 7, int(jobs), int(chunk))
        assert bits(got).tolist() == hex_to_bits(want["moments"]).tolist(), key
