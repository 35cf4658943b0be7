"""Production mode on the GPU (counter stream): bit-exact against the CPU oracle
and against the reference itself (golden ctr fixtures), plus edge cases."""
import numpy as np
import pytest

from helpers import assert_bits_equal, bits, hex_to_bits

pytestmark = pytest.mark.gpu

DISTS = ["exp", "normal"]


def sampler(zf, dist, seed, counter=0, device=None):
    cls = zf.ExpSampler if dist == "exp" else zf.NormalSampler
    return cls(source=zf.UniformSource.counter(seed, counter), device=device)


@pytest.fixture(scope="module")
def zf(cuda):
    import paper_1403_6870_b200 as zf
    return zf


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("n", [1, 2, 7, 31, 511, 512, 513, 4096, 100_003])
def test_fill_matches_oracle(zf, orc, cuda, dist, n):
    got = sampler(zf, dist, 1234, device=cuda).fill(n).cpu().numpy()
    want, _, _ = orc.fill_ctr(dist, n, seed=1234)
    assert_bits_equal(got, bits(want), f"{dist} n={n}")


@pytest.mark.parametrize("dist", DISTS)
def test_fill_matches_reference_replay(zf, golden, cuda, dist):
    """Golden values computed by the reference (replay of each sample's words)."""
    for key, want in golden[f"ctr_{dist}"].items():
        seed, base = (int(x) for x in key.split(":"))
        got = sampler(zf, dist, seed, base, device=cuda).fill(len(want)).cpu().numpy()
        assert_bits_equal(got, hex_to_bits(want), f"ctr {key}")


@pytest.mark.parametrize("dist", DISTS)
def test_large_counter_offsets(zf, orc, cuda, dist):
    for base in (1 << 40, 3 << 40, (1 << 44) - 10_000):
        got = sampler(zf, dist, 7, base, device=cuda).fill(10_000).cpu().numpy()
        want, _, _ = orc.fill_ctr(dist, 10_000, seed=7, ctr_base=base)
        assert_bits_equal(got, bits(want), f"base {base}")


def test_counter_range_enforced(zf, cuda):
    s = sampler(zf, "exp", 1, (1 << 44) - 5, device=cuda)
    with pytest.raises(ValueError):
        s.fill(10)


@pytest.mark.parametrize("dist", DISTS)
def test_stream_continuity(zf, cuda, dist):
    """fill(a); fill(b) == fill(a + b), and equals sample() repeated."""
    a = sampler(zf, dist, 99, device=cuda)
    first, second = a.fill(1000).cpu().numpy(), a.fill(2345).cpu().numpy()
    whole = sampler(zf, dist, 99, device=cuda).fill(3345).cpu().numpy()
    assert np.array_equal(bits(np.concatenate([first, second])), bits(whole))
    c = sampler(zf, dist, 99, device=cuda)
    singles = np.array([c.sample() for _ in range(20)])
    assert np.array_equal(bits(singles), bits(whole[:20]))


@pytest.mark.parametrize("dist", DISTS)
def test_float32_is_rounded_float64(zf, cuda, dist):
    import torch
    n = 50_001
    f64 = sampler(zf, dist, 5, device=cuda).fill(n)
    out = torch.empty(n, dtype=torch.float32, device=cuda)
    sampler(zf, dist, 5, device=cuda).fill(out)
    assert torch.equal(out, f64.to(torch.float32))


@pytest.mark.parametrize("dist", DISTS)
def test_misaligned_and_strided_views(zf, orc, cuda, dist):
    import torch
    buf = torch.zeros(10_001, dtype=torch.float64, device=cuda)
    view = buf[1:]  # 8-byte aligned only: scalar-store kernel variant
    sampler(zf, dist, 3, device=cuda).fill(view)
    want, _, _ = orc.fill_ctr(dist, 10_000, seed=3)
    assert_bits_equal(view.cpu().numpy(), bits(want))
    assert buf[0].item() == 0.0
    # strided views, device and host (the reference's kernels write out[k]
    # through any strides): values land in element order, the gaps untouched
    buf.zero_()
    r = sampler(zf, dist, 3, device=cuda).fill(buf[::2])
    assert r.data_ptr() == buf.data_ptr() and r.numel() == 5001
    want5, _, _ = orc.fill_ctr(dist, 5001, seed=3)
    assert_bits_equal(buf[::2].cpu().numpy(), bits(want5))
    assert not buf[1::2].any().item()
    host = np.zeros((300, 4))
    col = host[:, 1]
    assert sampler(zf, dist, 3, device=cuda).fill(col) is col
    assert_bits_equal(host[:, 1], bits(want5[:300]))
    assert not host[:, [0, 2, 3]].any()


@pytest.mark.parametrize("dist", DISTS)
def test_empty_fill(zf, cuda, dist):
    s = sampler(zf, dist, 3, device=cuda)
    assert s.fill(0).numel() == 0
    assert int(s.source.state[1]) == 0


@pytest.mark.parametrize("dist", DISTS)
def test_host_destinations(zf, orc, cuda, dist):
    import torch
    n = (1 << 24) + 77  # more than one host chunk
    want, _, _ = orc.fill_ctr(dist, n, seed=11)
    arr = np.zeros(n)
    out = sampler(zf, dist, 11, device=cuda).fill(arr)
    assert out is arr
    assert np.array_equal(bits(arr), bits(want))
    pinned = torch.empty(1000, dtype=torch.float64).pin_memory()
    sampler(zf, dist, 11, device=cuda).fill(pinned)
    assert np.array_equal(bits(pinned.numpy()), bits(want[:1000]))


@pytest.mark.parametrize("dist", DISTS)
def test_pageable_staging_paths(zf, cuda, dist, monkeypatch):
    """The pinned-staging route for pageable host memory (several staging
    chunks, ragged last one): fp32, counted fills, oracle-mode sources, CPU
    tensors and concurrent callers all equal the device-resident fill.
    (Registration in place is switched off here so the staging path runs.)"""
    import threading
    import torch
    from paper_1403_6870_b200 import samplers
    monkeypatch.setattr(samplers, "_REGISTER_MIN_BYTES", 1 << 62)
    n32 = 3 * (16 << 20) + 5
    a32 = np.empty(n32, dtype=np.float32)
    sampler(zf, dist, 5, device=cuda).fill(a32)
    d32 = torch.empty(n32, dtype=torch.float32, device=cuda)
    sampler(zf, dist, 5, device=cuda).fill(d32)
    assert np.array_equal(a32.view(np.uint32), d32.cpu().numpy().view(np.uint32))

    n = (17 << 20) + 3
    s_host, s_dev = sampler(zf, dist, 6, device=cuda), sampler(zf, dist, 6, device=cuda)
    host = torch.empty(n, dtype=torch.float64)
    s_host.fill_counted(host)
    want = s_dev.fill_counted(n)
    assert torch.equal(host, want.cpu())
    assert s_host.counters.tolist() == s_dev.counters.tolist()

    cls = zf.ExpSampler if dist == "exp" else zf.NormalSampler
    o_host, o_dev = (cls(source=zf.UniformSource(8), device=cuda) for _ in range(2))
    arr = np.empty(n)
    o_host.fill(arr)
    assert np.array_equal(bits(arr), bits(o_dev.fill(n).cpu().numpy()))
    assert np.array_equal(o_host.source.state, o_dev.source.state)

    outs = [np.empty(n) for _ in range(3)]
    ths = [threading.Thread(target=lambda k=k: sampler(zf, dist, 40 + k, device=cuda).fill(outs[k]))
           for k in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for k in range(3):
        ref = sampler(zf, dist, 40 + k, device=cuda).fill(n).cpu().numpy()
        assert np.array_equal(bits(outs[k]), bits(ref)), k


@pytest.mark.parametrize("dist", DISTS)
def test_counters_match_oracle(zf, orc, cuda, dist):
    s = sampler(zf, dist, 21, device=cuda)
    s.fill_counted(300_000)
    _, cnt, _ = orc.fill_ctr(dist, 300_000, seed=21)
    assert s.counters.tolist() == cnt.tolist()
    c = s.path_counts
    if dist == "exp":
        assert c.byte_draws == 300_000 + c.tail
        assert c.box_attempts == c.overhang_fast + c.band_evals
    else:
        assert c.byte_draws == 300_000
    s.reset_counters()
    assert s.path_counts.byte_draws == 0


def test_batch_matches_individual_fills(zf, orc, cuda):
    reqs = []
    for i in range(64):
        reqs.append(("exp" if i % 2 == 0 else "normal", 8192 if i % 5 else 1000 + i, i))
    out, offs = zf.fill_batch(reqs, device=cuda)
    host = out.cpu().numpy()
    for (dist, n, seed), off in zip(reqs, offs):
        want, _, _ = orc.fill_ctr(dist, n, seed=seed)
        assert np.array_equal(bits(host[off:off + n]), bits(want)), (dist, n, seed)


def test_batch_staging_ring_reuse(zf, orc, cuda):
    """Back-to-back batches on one tables handle without host syncs: the
    request tables go through the handle's reused pinned/device staging slots
    (which grow with the batch), so every batch must still see its own table."""
    import torch
    batches, outs = [], []
    for b, m in enumerate((3, 40, 7, 300, 300, 12)):  # grows, shrinks, grows past capacity
        reqs = [("normal" if (i + b) % 3 else "exp", 700 + 97 * i, 1000 * b + i) for i in range(m)]
        out, offs = zf.fill_batch(reqs, device=cuda)  # no synchronize between batches
        batches.append((reqs, offs))
        outs.append(out)
    torch.cuda.synchronize(cuda)
    for (reqs, offs), out in zip(batches, outs):
        host = out.cpu().numpy()
        for (dist, n, seed), off in zip(reqs[::17], offs[::17]):
            want, _, _ = orc.fill_ctr(dist, n, seed=seed)
            assert np.array_equal(bits(host[off:off + n]), bits(want)), (dist, n, seed)


def test_batch_plan_resident_refills(zf, orc, cuda):
    """A BatchPlan keeps its request table on the device (zf_batch_create):
    refills are single launches; every refill (into fresh and reused outputs)
    equals the individual fills."""
    import torch
    reqs = [("exp" if i % 2 else "normal", 8192 if i % 7 else 3000 + i, 50 + i) for i in range(97)]
    plan = zf.BatchPlan([r[0] for r in reqs], [r[1] for r in reqs], [r[2] for r in reqs])
    first = plan.fill(device=cuda).cpu().numpy()
    again = torch.full((plan.total,), float("nan"), dtype=torch.float64, device=cuda)
    for _ in range(3):
        plan.fill(out=again, device=cuda)
    host = again.cpu().numpy()
    for (_, n, _), off in zip(reqs, plan.offsets):  # (padding between requests is not written)
        assert np.array_equal(bits(first[off:off + n]), bits(host[off:off + n]))
    for (dist, n, seed), off in zip(reqs, plan.offsets):
        want, _, _ = orc.fill_ctr(dist, n, seed=seed)
        assert np.array_equal(bits(host[off:off + n]), bits(want)), (dist, n, seed)


def test_production_launches_capture_into_cuda_graphs(zf, orc, cuda):
    """`zf_fill` (fp64, fp32) and `zf_batch_fill` are plain launches on the caller's
    stream -- no allocation, synchronisation or host round trip -- so a
    launch-bound inner loop can live in a CUDA graph ("batch
    into one launch/graph").  A replay redoes the captured (seed, counter)
    ranges: the graph's outputs equal the oracle after every replay."""
    import torch
    n = 200_003
    outs = {d: torch.empty(n, dtype=torch.float64, device=cuda) for d in DISTS}
    f32 = torch.empty(n, dtype=torch.float32, device=cuda)
    reqs = [("exp" if i % 2 else "normal", 8192, 900 + i) for i in range(64)]
    plan = zf.BatchPlan([r[0] for r in reqs], [r[1] for r in reqs], [r[2] for r in reqs])
    bout = torch.empty(plan.total, dtype=torch.float64, device=cuda)
    plan.fill(out=bout, device=cuda)  # the plan's device image exists before the capture
    samplers = {d: sampler(zf, d, 77, 1 << 40, device=cuda) for d in DISTS}
    s32 = sampler(zf, "normal", 78, device=cuda)
    torch.cuda.synchronize(cuda)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for d in DISTS:
            samplers[d].fill(outs[d])
        s32.fill(f32)
        plan.fill(out=bout, device=cuda)
    for rep in range(3):
        for t in (*outs.values(), f32, bout):
            t.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize(cuda)
        for d in DISTS:
            want, _, _ = orc.fill_ctr(d, n, seed=77, ctr_base=1 << 40)
            assert_bits_equal(outs[d].cpu().numpy(), bits(want), f"graph {d} replay {rep}")
        want, _, _ = orc.fill_ctr("normal", n, seed=78)
        assert np.array_equal(f32.cpu().numpy(), want.astype(np.float32))
        host = bout.cpu().numpy()
        for (dist, m, seed), off in zip(reqs, plan.offsets):
            want, _, _ = orc.fill_ctr(dist, m, seed=seed)
            assert np.array_equal(bits(host[off:off + m]), bits(want)), (dist, seed, rep)
    # the samplers' host-side counters advanced once, at capture time
    assert int(samplers["exp"].source.state[1]) == (1 << 40) + n


def test_convenience_api(zf, cuda):
    zf.seed(2024)
    a = zf.normal(1000, device=cuda)
    b = zf.normal(500, device=cuda)
    zf.seed(2024)
    c = zf.normal(1500, device=cuda)
    assert np.array_equal(bits(np.concatenate([a.cpu().numpy(), b.cpu().numpy()])),
                          bits(c.cpu().numpy()))
    assert zf.standard_exponential(10, device=cuda).min().item() > 0.0


@pytest.mark.parametrize("dist", DISTS)
def test_full_size_fill_properties(zf, orc, cuda, dist):
    """BASELINE config 3 size on one GPU (n = 2^32 + 77, 32 GiB): spot-check
    windows against the oracle at arbitrary offsets, and size-independent
    properties (finite, sign/positivity, moments within 6 sigma)."""
    import torch
    from paper_1403_6870_b200 import quality
    n = (1 << 32) + 77
    free, _ = torch.cuda.mem_get_info(cuda)
    if free < 8 * n + (4 << 30):
        pytest.skip("not enough device memory")
    s = sampler(zf, dist, 7, 1 << 40, device=cuda)
    out = s.fill(n)
    for off in (0, 12345, (1 << 31) + 3, n - 1000):
        want, _, _ = orc.fill_ctr(dist, 1000, seed=7, ctr_base=(1 << 40) + off)
        assert np.array_equal(bits(out[off:off + 1000].cpu().numpy()), bits(want)), off
    sums, res = quality.buffer_sums(out, thresholds=(0.0,))
    raw = [v / n for v in sums]
    if dist == "normal":
        mean, var, skew, exk = quality.central_moments_from_raw(raw)
        for val, se in ((mean, (1 / n) ** 0.5), (var - 1, (2 / n) ** 0.5),
                        (skew, (6 / n) ** 0.5), (exk, (24 / n) ** 0.5)):
            assert abs(val / se) < 6.0
        assert abs(res.thresh_counts[0] - n / 2) < 6 * (n / 4) ** 0.5
    else:
        assert res.thresh_counts[0] == n  # every draw > 0
        for k, want in enumerate((1.0, 2.0)):
            sd = quality._MOMENT_SD["exp"][k] / n ** 0.5
            assert abs(raw[k] - want) < 6 * sd
    assert torch.isfinite(out).all().item()
    del out
    torch.cuda.empty_cache()


def test_concurrent_host_threads(zf, orc, cuda):
    """Samplers are single-owner, the uploaded tables are shared: several host
    threads filling on their own streams give the same bits as serial fills."""
    import threading

    import torch
    results = {}

    def work(i):
        st = torch.cuda.Stream(cuda)
        with torch.cuda.stream(st):
            s = sampler(zf, "normal" if i % 2 else "exp", 100 + i, device=cuda)
            v = s.fill(200_000)
        st.synchronize()
        results[i] = v.cpu().numpy()

    threads = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for i in range(6):
        want, _, _ = orc.fill_ctr("normal" if i % 2 else "exp", 200_000, seed=100 + i)
        assert np.array_equal(bits(results[i]), bits(want)), i


@pytest.mark.parametrize("dist", DISTS)
def test_scalar_samples_interleave_with_fills(zf, cuda, dist):
    """sample() serves production draws from a cached block but advances the
    stream by one per call: any interleaving of sample() and fill() equals one
    long fill, and an external counter change invalidates the block."""
    whole = sampler(zf, dist, 31, device=cuda).fill(9000).cpu().numpy()
    s = sampler(zf, dist, 31, device=cuda)
    got = [s.sample() for _ in range(3)]
    got += list(s.fill(100).cpu().numpy())
    got += [s.sample() for _ in range(5000)]  # crosses a cache block
    got += list(s.fill(7).cpu().numpy())
    got += [s.sample() for _ in range(2)]
    assert np.array_equal(bits(np.array(got)), bits(whole[:len(got)]))
    s.source.state[1] = np.uint64(5)  # rewind: the cached block must not be reused blindly
    assert bits(np.array([s.sample()]))[0] == bits(whole[5:6])[0]


def test_batch_fp32_and_counter_bases(zf, orc, cuda):
    """fp32 batches (4-element alignment padding) and nonzero counter bases."""
    import torch
    dists = ["exp", "normal", "normal", "exp", "exp"]
    ns = [1, 511, 4097, 20000, 3]
    seeds = [5, 6, 7, 8, 9]
    bases = [0, 1 << 40, 123, (1 << 44) - 30000, 77]
    plan = zf.BatchPlan(dists, ns, seeds, bases, dtype="float32")
    out = plan.fill(device=cuda).cpu().numpy()
    for d, n, sd, b, off in zip(dists, ns, seeds, bases, plan.offsets):
        want, _, _ = orc.fill_ctr(d, n, seed=sd, ctr_base=b)
        assert np.array_equal(out[off:off + n], want.astype(np.float32)), (d, n, sd, b)


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("shift", [1, 2, 3])
def test_misaligned_fp32_views(zf, orc, cuda, dist, shift):
    """fp32 outputs 4-byte aligned but not 16: the scalar-store kernel variant."""
    import torch
    buf = torch.zeros(5003, dtype=torch.float32, device=cuda)
    view = buf[shift:shift + 4000]
    sampler(zf, dist, 13, device=cuda).fill(view)
    want, _, _ = orc.fill_ctr(dist, 4000, seed=13)
    assert np.array_equal(view.cpu().numpy(), want.astype(np.float32))
    assert buf[:shift].abs().sum().item() == 0.0 and buf[shift + 4000:].abs().sum().item() == 0.0


def test_pageable_numpy_fill_page_locks_in_place(zf, cuda):
    """fill(np.empty(n)) -- the reference's usage -- page-locks a large array
    once (cached while it lives, unregistered when it is collected) and DMAs
    into it; values equal the device fill, views of a registered array too."""
    import gc
    from paper_1403_6870_b200 import samplers
    n = 1 << 24  # 128 MiB, above the registration threshold
    arr = np.empty(n)
    a = zf.NormalSampler(source=zf.UniformSource.counter(31, 77), device=cuda)
    a.fill(arr)
    want = zf.NormalSampler(source=zf.UniformSource.counter(31, 77), device=cuda).fill(n)
    assert np.array_equal(arr.view(np.uint64), want.cpu().numpy().view(np.uint64))
    ptr = arr.ctypes.data
    assert ptr in samplers._registered
    view = arr[1000:1000 + (1 << 23)]  # a view: its owner is already registered
    b = zf.ExpSampler(source=zf.UniformSource.counter(5), device=cuda)
    b.fill(view)
    wv = zf.ExpSampler(source=zf.UniformSource.counter(5), device=cuda).fill(1 << 23)
    assert np.array_equal(view.view(np.uint64), wv.cpu().numpy().view(np.uint64))
    assert arr[999] == want[999].item()  # untouched outside the view
    del arr, view
    gc.collect()
    assert ptr not in samplers._registered
    # small arrays take the staged path and are not registered
    small = np.empty(1 << 16)
    a.fill(small)
    assert small.ctypes.data not in samplers._registered


@pytest.mark.parametrize("dist", DISTS)
def test_full_comparison_many_tiles_per_warp(zf, orc, cuda, dist):
    """n = 2^26 against the oracle in fp64 and fp32: each warp walks ~9 tiles,
    so the cross-tile paths (the per-warp queue carried over tiles, rounds of
    32 from several tiles, queue compaction, cooperative normal rounds) all
    run many times."""
    import torch
    n = 1 << 26
    want, _, _ = orc.fill_ctr(dist, n, seed=4242, ctr_base=1 << 41)
    got = sampler(zf, dist, 4242, 1 << 41, device=cuda).fill(n).cpu().numpy()
    assert_bits_equal(got, bits(want), f"{dist} f64 2^26")
    g32 = torch.empty(n, dtype=torch.float32, device=cuda)
    sampler(zf, dist, 4242, 1 << 41, device=cuda).fill(g32)
    assert np.array_equal(g32.cpu().numpy().view(np.uint32), want.astype(np.float32).view(np.uint32))


_WAVES_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import torch
import paper_1403_6870_b200 as zf
for cls in (zf.ExpSampler, zf.NormalSampler):
    x = cls(source=zf.UniformSource.counter(77, 5), device="cuda").fill(1 << 24)
    print(hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest())
"""


def test_one_wave_grid_many_tiles_per_warp(orc, cuda):
    """ZF_GRID_WAVES=1 in a fresh process: one resident wave, so every warp
    carries its queue across ~16 tiles of a 2^24 fill; bit-exact with the
    oracle."""
    import hashlib
    import os
    import pathlib
    import subprocess
    import sys
    root = str(pathlib.Path(__file__).resolve().parents[1])
    env = dict(os.environ, ZF_GRID_WAVES="1")
    res = subprocess.run([sys.executable, "-c", _WAVES_SCRIPT, root], env=env,
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    got = res.stdout.split()
    for dist, h in zip(("exp", "normal"), got):
        want, _, _ = orc.fill_ctr(dist, 1 << 24, seed=77, ctr_base=5)
        assert h == hashlib.sha256(want.tobytes()).hexdigest(), dist
