"""Oracle mode on the GPU: the reference's own sequential streams (xoshiro256++,
splitmix64, replay) resolved in parallel; bit-exact values AND path records."""
import hashlib

import numpy as np
import pytest

from helpers import assert_bits_equal, bits, hex_to_bits

pytestmark = pytest.mark.gpu

DISTS = ["exp", "normal"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def zf(cuda):
    import paper_1403_6870_b200 as zf
    return zf


def cls_of(zf, dist):
    return zf.ExpSampler if dist == "exp" else zf.NormalSampler


def test_xoshiro_words_on_device(zf, golden, cuda):
    src = zf.UniformSource(12345)
    assert [int(w) for w in src.next_block(8)] == golden["xoshiro_12345_first8"]
    src = zf.UniformSource(42)
    words = src.next_block(1_100_000)
    assert sha(words) == golden["xoshiro_42_1p1M_sha256"]
    # block then scalar continues the stream (reference test_uniform.py:136-142)
    a, b = zf.UniformSource(7), zf.UniformSource(7)
    a.next_block(13)
    b.next_block(5)
    b.next_block(8)
    assert a.next_u64() == b.next_u64()


def test_jump_matches_golden_state(zf, golden):
    src = zf.UniformSource(42)
    src.jump(1_000_000)
    assert [format(int(w), "016x") for w in src.state] == golden["xoshiro_42_after_1M_state"]


@pytest.mark.parametrize("dist", DISTS)
def test_seed7_golden(zf, golden, cuda, dist):
    s = cls_of(zf, dist)(source=zf.UniformSource(7), device=cuda)
    first = [s.sample() for _ in range(5)]
    assert_bits_equal(first, hex_to_bits(golden[f"{dist}_seed7_first5"]))
    got = cls_of(zf, dist)(source=zf.UniformSource(7), device=cuda).fill(3000).cpu().numpy()
    assert_bits_equal(got, hex_to_bits(golden[f"{dist}_seed7_fill3000"]))
    got = cls_of(zf, dist)(source=zf.UniformSource(99, generator="splitmix64"),
                           device=cuda).fill(2000).cpu().numpy()
    assert_bits_equal(got, hex_to_bits(golden[f"{dist}_splitmix99_fill2000"]))


@pytest.mark.parametrize("dist", DISTS)
def test_fill_equals_repeated_samples(zf, cuda, dist):
    a = cls_of(zf, dist)(source=zf.UniformSource(7), device=cuda)
    b = cls_of(zf, dist)(source=zf.UniformSource(7), device=cuda)
    block = a.fill(300).cpu().numpy()
    singles = np.array([b.sample() for _ in range(300)])
    assert np.array_equal(bits(block), bits(singles))
    # and the host state advanced identically
    assert np.array_equal(a.source.state, b.source.state)


def test_replay_known_answers(zf, golden, cuda):
    w = golden["kat_word"]
    U = zf.UniformSource
    assert_bits_equal([zf.ExpSampler(source=U.replay([w]), device=cuda).sample()],
                      hex_to_bits(golden["kat_exp_common"]))
    assert_bits_equal([zf.ExpSampler(source=U.replay([255, 0, 0, w]), device=cuda).sample()],
                      hex_to_bits(golden["kat_exp_tail"]))
    assert_bits_equal([zf.NormalSampler(source=U.replay([w]), device=cuda).sample()],
                      hex_to_bits(golden["kat_normal_common"]))
    assert_bits_equal([zf.NormalSampler(source=U.replay([(1 << 63) | w]), device=cuda).sample()],
                      hex_to_bits(golden["kat_normal_neg"]))


@pytest.mark.parametrize("dist", DISTS)
def test_replay_wraps_like_reference(zf, golden, cuda, dist):
    s = cls_of(zf, dist)(source=zf.UniformSource.replay(hex_to_bits(golden["wrap_words"])),
                         device=cuda)
    got = s.fill(40).cpu().numpy()
    assert_bits_equal(got, hex_to_bits(golden[f"{dist}_wrap_fill40"]))
    assert int(s.source.state[0]) == golden[f"{dist}_wrap_cursor"]


@pytest.mark.parametrize("dist", DISTS)
def test_config1_bit_exact_with_paths(zf, golden, cuda, dist):
    """BASELINE config 1: n = 1e6 from UniformSource(42).  Values, counters,
    words consumed and every per-sample path record equal the reference's."""
    g = golden[f"c1_{dist}"]
    s = cls_of(zf, dist)(source=zf.UniformSource(42), device=cuda)
    vals, recs = s.fill_records(g["n"])
    vals = vals.cpu().numpy()
    assert_bits_equal(vals[:64], hex_to_bits(g["head"]), "head")
    assert_bits_equal(vals[-64:], hex_to_bits(g["tail"]), "tail")
    assert sha(vals) == g["values_sha256"]
    assert sha(recs["start"]) == g["starts_sha256"]
    assert sha(recs["nwords"]) == g["nwords_sha256"]
    assert sha(recs["layer"]) == g["layer_sha256"]
    assert sha(recs["path"]) == g["path_sha256"]
    if g["attempts_sha256"]:
        assert sha(recs["attempts"]) == g["attempts_sha256"]
    # box attempts of every non-tail sample (the reference's slot 5 counts box
    # attempts only; our record counts tail rounds for tail samples)
    att_box = np.where(recs["path"] & 2, 0, recs["attempts"]).astype(np.uint16)
    assert sha(att_box) == g["attempts_box_sha256"]
    c = cls_of(zf, dist)(source=zf.UniformSource(42), device=cuda)
    c.fill_counted(g["n"])
    assert c.counters.tolist() == g["counters"]
    ref_state = zf.UniformSource(42)
    ref_state.jump(g["words_consumed"])
    assert np.array_equal(c.source.state, ref_state.state)


@pytest.mark.parametrize("dist", DISTS)
def test_records_match_oracle(zf, orc, cuda, dist):
    n = 200_000
    s = cls_of(zf, dist)(source=zf.UniformSource(2024, generator="splitmix64"), device=cuda)
    vals, recs = s.fill_records(n)
    want, _, wrecs, _ = orc.fill_stream(dist, n, generator="splitmix64", seed=2024, records=True)
    assert np.array_equal(bits(vals.cpu().numpy()), bits(want))
    for f in ("start", "nwords", "layer", "path", "attempts"):
        assert np.array_equal(recs[f], wrecs[f]), f


@pytest.mark.parametrize("dist", DISTS)
def test_replay_cursor_continues(zf, orc, cuda, dist):
    words = orc.words("xoshiro256++", 5, 50_000)
    s = cls_of(zf, dist)(source=zf.UniformSource.replay(words), device=cuda)
    a = s.fill(10_000).cpu().numpy()
    b = s.fill(20_000).cpu().numpy()
    want, _, _, used = orc.fill_stream(dist, 30_000, replay_words=words)
    assert np.array_equal(bits(np.concatenate([a, b])), bits(want))
    assert int(s.source.state[0]) == used


@pytest.mark.parametrize("dist", DISTS)
def test_long_stream_many_windows(zf, orc, cuda, dist):
    """A fill large enough to need several replay windows (grow + retry)."""
    n = 3_000_000
    got = cls_of(zf, dist)(source=zf.UniformSource(77), device=cuda).fill(n).cpu().numpy()
    want, _, _, _ = orc.fill_stream(dist, n, seed=77)
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("dist", DISTS)
def test_config2_sized_stream_every_sample(zf, orc, cuda, dist):
    """The reference's own xoshiro256++ stream at BASELINE config 2's size
    (n = 2^28, 2 GiB): every sample of one `fill` against the sequential CPU
    oracle, then the stream continues where the reference's would."""
    n = 1 << 28
    seed = orc.derive_seed(1234, 0)  # what fill_sharded's only thread seeds with
    s = cls_of(zf, dist)(source=zf.UniformSource(seed), device=cuda)
    got = s.fill(n).cpu().numpy()
    tail = s.fill(1000).cpu().numpy()
    want = orc.fill_sharded(dist, n + 1000, 1234, threads=1)
    diff = np.flatnonzero(bits(got) != bits(want[:n]))
    assert diff.size == 0, f"{diff.size} mismatches, first at {int(diff[0])}"
    assert np.array_equal(bits(tail), bits(want[n:]))


def test_fill_above_one_window_continues_the_stream(zf, orc, cuda):
    """A single oracle-mode fill larger than the C-ABI's 2^28-sample window
    chunk (the reference has no size limit): the chunks continue one stream --
    checked on the chunk boundary, the end, the continuation and the counters
    of a counted fill against the sequential oracle."""
    n = (1 << 28) + 1_000_003
    seed = orc.derive_seed(5, 0)
    s = zf.ExpSampler(source=zf.UniformSource(seed), device=cuda)
    got = s.fill_counted(n)
    tail = s.fill(512).cpu().numpy()
    want = orc.fill_sharded("exp", n + 512, 5, threads=1)
    for lo, hi in ((0, 4096), ((1 << 28) - 4096, (1 << 28) + 4096), (n - 4096, n)):
        assert np.array_equal(bits(got[lo:hi].cpu().numpy()), bits(want[lo:hi])), lo
    assert np.array_equal(bits(tail), bits(want[n:]))
    _, cnt, _, _ = orc.fill_stream("exp", n, seed=seed)
    assert s.path_counts.as_tuple() == tuple(int(v) for v in cnt)


def test_fill_of_more_than_2p31_samples(zf, orc, cuda):
    """n above the 32-bit window positions (the old ZF_ERANGE): the last sample
    of a 2^31 + 5 sample N(0,1) fill equals the sequential oracle's (which
    keeps only a small buffer), so all eight chunks consumed the right words."""
    import torch
    n = (1 << 31) + 5
    free, _ = torch.cuda.mem_get_info(cuda)
    if free < 8 * n + (8 << 30):
        pytest.skip("not enough device memory")
    seed = orc.derive_seed(11, 0)
    out = zf.NormalSampler(source=zf.UniformSource(seed), device=cuda).fill(n)
    last = out[-1].item()
    first = out[:1000].cpu().numpy()
    del out
    torch.cuda.empty_cache()
    assert bits(np.array([last]))[0] == bits(np.array([orc.fill_sharded_chunked(
        "normal", n, 11, threads=1)]))[0]
    assert np.array_equal(bits(first), bits(orc.fill_sharded("normal", 1000, 11, threads=1)))


def test_adversarial_replay_all_exceptional(zf, orc, cuda):
    """Every word exceptional (byte 255): long overlapping draw chains."""
    rng = np.random.default_rng(0)
    words = (rng.integers(0, 2**63, 5000, dtype=np.uint64) << np.uint64(8)) | np.uint64(0xFF)
    words[::7] &= ~np.uint64(0xFF)  # sprinkle a few common-path words
    for dist in DISTS:
        s = cls_of(zf, dist)(source=zf.UniformSource.replay(words), device=cuda)
        got = s.fill(3000).cpu().numpy()
        want, _, _, used = orc.fill_stream(dist, 3000, replay_words=words)
        assert np.array_equal(bits(got), bits(want)), dist
        assert int(s.source.state[0]) == used


@pytest.mark.parametrize("frac", [0.9, 0.07, 0.04])
def test_replay_exceptional_count_above_the_bound(zf, orc, cuda, frac):
    """The exceptional arrays are sized for a bound (6.25 % of the window +
    4096) without a host round trip; windows with more exceptional words (90 %)
    are redone with exact sizes, windows near the bound (7 %, 4 %) pass
    either way.  Values and words consumed equal the reference's."""
    rng = np.random.default_rng(int(frac * 100))
    m = 400_000
    words = rng.integers(0, 2**63, m, dtype=np.uint64) << np.uint64(8)
    exc = rng.random(m) < frac
    words[exc] |= np.uint64(0xFF)
    words[~exc] |= rng.integers(0, 200, int((~exc).sum()), dtype=np.uint64)
    for dist in DISTS:
        s = cls_of(zf, dist)(source=zf.UniformSource.replay(words), device=cuda)
        got = s.fill(100_000).cpu().numpy()
        want, _, _, used = orc.fill_stream(dist, 100_000, replay_words=words)
        assert np.array_equal(bits(got), bits(want)), dist
        assert int(s.source.state[0]) == used


def test_cycling_replay_is_an_error_not_a_hang(zf, cuda):
    """A short wrapping list on which a normal-tail draw can never finish (the
    reference would loop forever) fails with ZF_ERANGE instead of hanging."""
    from paper_1403_6870_b200.errors import DeviceError
    s = zf.NormalSampler(source=zf.UniformSource.replay([255, 0, 0, 123456789 << 8, 7]),
                         device=cuda)
    with pytest.raises(DeviceError) as ei:
        s.fill(100)
    assert ei.value.status == -4


@pytest.mark.parametrize("dist", DISTS)
def test_scalar_samples_interleave_with_fills(zf, orc, cuda, dist):
    """sample() on a reference stream serves a cached block of draws but
    advances the source by exactly each draw's words: interleaving sample()
    and fill() equals one fill, with the reference's state at every point."""
    want, _, _, _ = orc.fill_stream(dist, 6000, seed=5)
    s = cls_of(zf, dist)(source=zf.UniformSource(5), device=cuda)
    got = [s.sample() for _ in range(10)]
    got += list(s.fill(500).cpu().numpy())
    got += [s.sample() for _ in range(4200)]  # crosses a cached block
    got += list(s.fill(3).cpu().numpy())
    assert np.array_equal(bits(np.array(got)), bits(want[:len(got)]))
    ref = zf.UniformSource(5)
    _, _, _, used = orc.fill_stream(dist, len(got), seed=5)
    ref.jump(used)
    assert np.array_equal(s.source.state, ref.state)
    # an outside reseed invalidates the cached block
    s.source.state[:] = zf.UniformSource(5).state
    assert bits(np.array([s.sample()]))[0] == bits(want[:1])[0]


def test_scalar_sample_before_a_cycling_draw(zf, golden, cuda):
    """Replay list [255, 0, 0, w, 7] read from cursor 3: two fast draws, then
    the wrap reaches a normal-tail draw that never finishes.  The block resolve
    fails, sample() falls back to single draws on the real source: the first
    two values come back with the cursor advanced, the third raises (the
    reference would hang on it)."""
    from paper_1403_6870_b200.errors import DeviceError
    w = golden["kat_word"]
    s = zf.NormalSampler(source=zf.UniformSource.replay([255, 0, 0, w, 7]), device=cuda)
    s.source.state[0] = np.uint64(3)
    assert_bits_equal([s.sample()], hex_to_bits(golden["kat_normal_common"]))
    assert int(s.source.state[0]) == 4
    s.sample()
    assert int(s.source.state[0]) == 5
    with pytest.raises(DeviceError):
        s.sample()
