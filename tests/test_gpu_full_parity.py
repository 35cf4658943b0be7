"""BASELINE config 3 in full: EVERY sample of a 2^32-sample production fill --
one launch, the grid shape the bench times -- compared bit for bit with the CPU
oracle (`oracle.check_ctr`: the reference's draw body, _kernels.py:149-181 and
:406-495, over each sample's own word list, on all host threads, in place).
The output leaves the device in 2^27-sample chunks through two pinned buffers,
the copy of chunk i+1 overlapping the check of chunk i."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CHUNK = 1 << 27


def _check_whole(zf, orc, cuda, dist, dtype, n, seed, base, corrupt=()):
    """Returns (mismatches, lowest mismatching index); `corrupt`: sample indices
    whose lowest bit is flipped on the device after the fill (negative control)."""
    import torch
    free, _ = torch.cuda.mem_get_info(cuda)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    esz = 8 if dtype == "f64" else 4
    if free < esz * n + (2 << 30):
        pytest.skip("not enough device memory")
    cls = zf.ExpSampler if dist == "exp" else zf.NormalSampler
    s = cls(source=zf.UniformSource.counter(seed, base), device=cuda)
    out = torch.empty(n, dtype=tdt, device=cuda)
    s.fill(out)  # ONE launch over the whole range
    if corrupt:
        idx = torch.tensor(list(corrupt), device=cuda)
        ints = out.view(torch.int64 if dtype == "f64" else torch.int32)
        ints[idx] ^= 1
    pinned = [torch.empty(min(CHUNK, n), dtype=tdt).pin_memory() for _ in range(2)]
    copy = torch.cuda.Stream(cuda)
    copy.wait_stream(torch.cuda.current_stream(cuda))
    events = [None, None]

    def start(i):
        off = i * CHUNK
        m = min(CHUNK, n - off)
        with torch.cuda.stream(copy):
            pinned[i & 1][:m].copy_(out[off:off + m], non_blocking=True)
            events[i & 1] = torch.cuda.Event()
            events[i & 1].record(copy)

    nchunks = (n + CHUNK - 1) // CHUNK
    start(0)
    bad_total, first_bad = 0, None
    for i in range(nchunks):
        events[i & 1].synchronize()
        if i + 1 < nchunks:
            start(i + 1)
        off = i * CHUNK
        m = min(CHUNK, n - off)
        bad, first = orc.check_ctr(dist, pinned[i & 1][:m].numpy(), seed, base + off)
        if bad and first_bad is None:
            first_bad = off + first
        bad_total += bad
    del out
    torch.cuda.empty_cache()
    return bad_total, first_bad


def _full_n():
    # ~1.3 G samples/s on 16 host threads; keep the check to seconds on small hosts
    return 1 << 32 if len(os.sched_getaffinity(0)) >= 8 else 1 << 29


@pytest.fixture(scope="module")
def zf(cuda):
    import paper_1403_6870_b200 as zf
    return zf


def test_config3_normal_every_sample(zf, orc, cuda):
    """Config 3 itself: N(0,1) fp64, n = 2^32, seed 7, GPU 0's counter range."""
    assert _check_whole(zf, orc, cuda, "normal", "f64", _full_n(), 7, 0) == (0, None)


def test_config3_rank1_exp_every_sample(zf, orc, cuda):
    """The exponential at the same size on GPU 1's counter range (base 2^40),
    ragged by 77 samples."""
    assert _check_whole(zf, orc, cuda, "exp", "f64", _full_n() + 77, 7, 1 << 40) == (0, None)


def test_fp32_normal_every_sample(zf, orc, cuda):
    """fp32 output (the fp64 draw rounded once), 2^31 samples."""
    assert _check_whole(zf, orc, cuda, "normal", "f32", min(_full_n(), 1 << 31), 7,
                        3 << 40) == (0, None)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_the_check_sees_single_bit_flips(zf, orc, cuda, dtype):
    """Negative control: three samples of a 2^29-sample fill with their lowest
    bit flipped on the device (first chunk, a chunk boundary, the last sample)
    are the only mismatches reported."""
    n = (1 << 29) + 5
    flips = (CHUNK - 1, 3 * CHUNK, n - 1)
    assert _check_whole(zf, orc, cuda, "normal", dtype, n, 99, 0, corrupt=flips) == (3, CHUNK - 1)


def test_config5_share_counts_equal_the_oracle(zf, orc, cuda):
    """BASELINE config 5, one GPU's share at 8 GPUs (2^33 N(0,1) + 2^33 Exp(1)
    draws, seed 99, rank 3's counter range): the in-kernel tail counts
    (|x| > 5, 6, 7; x > X[1]) equal the CPU oracle's over the same draws."""
    from paper_1403_6870_b200 import scale, shard
    from paper_1403_6870_b200.tables import default_tables
    m = _full_n() * 2
    base = shard.counter_base(3)
    x1 = float(default_tables("exponential").x[1])
    got_n = scale.device_counts("normal", scale.C5_SEED, base, m, scale.C5_THRESH, True,
                                device=cuda)
    got_e = scale.device_counts("exp", scale.C5_SEED, base, m, (x1,), False, device=cuda)
    assert [int(c) for c in got_n] == orc.count_ctr("normal", m, scale.C5_SEED, base,
                                                   scale.C5_THRESH, True)
    assert [int(c) for c in got_e] == orc.count_ctr("exp", m, scale.C5_SEED, base, (x1,), False)
