"""The N>1 host path on CPU: world_size 2 over gloo.  Each rank draws its
disjoint counter shard (with the CPU oracle standing in for the GPU kernel,
which the -m gpu tests pin bit-for-bit), then only validation statistics are
allreduced -- the same code bench.py runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from oracle import oracle
    from paper_1403_6870_b200 import shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base = shard.counter_base(rank)
    vals, cnt, _ = oracle.fill_ctr("normal", n, seed=7, ctr_base=base)
    sums = [float(np.sum(vals ** k)) for k in range(1, 6)]
    hist, _ = np.histogram(vals, bins=16, range=(-4.0, 4.0))
    tails = [int((np.abs(vals) > t).sum()) for t in (2.0, 3.0)]
    red = shard.allreduce_stats(shard.pack_stats(sums, hist, tails))
    rs, rh, rt = shard.unpack_stats(red, 5, 16, 2)
    out_q.put((rank, vals[:8].tobytes(), rs, rh, rt))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_and_stats_allreduce():
    from oracle import oracle
    from paper_1403_6870_b200 import shard
    world, n = 2, 20_000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank got identical reduced statistics
    assert res[0][2:] == res[1][2:]
    # which equal the statistics of the concatenated shards computed in one place
    allv = np.concatenate([oracle.fill_ctr("normal", n, seed=7, ctr_base=shard.counter_base(r))[0]
                           for r in range(world)])
    for k in range(5):
        assert res[0][2][k] == pytest.approx(float(np.sum(allv ** (k + 1))), rel=1e-12)
    assert res[0][3] == np.histogram(allv, bins=16, range=(-4.0, 4.0))[0].tolist()
    assert res[0][4] == [int((np.abs(allv) > t).sum()) for t in (2.0, 3.0)]
    # shards are the global stream at the rank offsets (independent of world size)
    for r, head, *_ in res:
        want = oracle.fill_ctr("normal", 8, seed=7, ctr_base=r << 40)[0]
        assert np.frombuffer(head, dtype=np.float64).tobytes() == want.tobytes()


def test_counter_base_range():
    from paper_1403_6870_b200 import shard
    assert shard.counter_base(3, 5) == 3 * 2**40 + 5
    with pytest.raises(ValueError):
        shard.counter_base(16)
    with pytest.raises(ValueError):
        shard.counter_base(0, 2**40)


def _oracle_counts(dist, seed, ctr_base, n, thresholds, abs_thresh):
    """CPU stand-in for scale.device_counts (the kernel call), same stream."""
    from oracle import oracle
    v = oracle.fill_ctr(dist, n, seed=seed, ctr_base=ctr_base)[0]
    a = np.abs(v) if abs_thresh else v
    return [int((a > t).sum()) for t in thresholds]


def _scale_worker(rank, world, port, total, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from oracle import oracle
    from paper_1403_6870_b200 import scale, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # config 5 with the kernel call stubbed by the oracle; thresholds low
    # enough that the small shares have tail counts to reduce
    rep5 = scale.config5(total, rank, world, stats=_oracle_counts, seed=99, exp_x1=2.0)
    # config 3 validation of this rank's shard
    m = scale.share(total, rank, world)
    v = oracle.fill_ctr("normal", m, seed=scale.C3_SEED, ctr_base=shard.counter_base(rank))[0]
    sums = [float(np.sum(v ** k)) for k in range(1, 6)]
    edges = np.linspace(-6.0, 6.0, 1025)
    h = np.histogram(v, bins=edges)[0]
    hist = [int((v < -6.0).sum())] + h.tolist() + [int((v >= 6.0).sum())]
    tails = [int((np.abs(v) > t).sum()) for t in scale.C3_THRESH]
    rep3 = scale.validate_config3(sums, hist, tails, m)
    out_q.put((rank, rep5, rep3))
    dist.barrier()
    dist.destroy_process_group()


def test_scale_configs_two_ranks():
    """bench.py's config-5 leg and config-3 validation at world size 2 (gloo):
    shares, counter bases and the allreduced counts equal a single-process
    computation over the concatenated shards."""
    from oracle import oracle
    from paper_1403_6870_b200 import scale, shard
    world, total = 2, 30_001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_scale_worker, args=(r, world, port, total, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1]["normal_abs_tails"] == res[1][1]["normal_abs_tails"]
    assert [scale.share(total, r, world) for r in range(world)] == [15001, 15000]
    # single-process reference: the two shards at their counter bases
    want_n = [0, 0, 0]
    want_e = 0
    allv = []
    for r in range(world):
        m = scale.share(total, r, world)
        vn = oracle.fill_ctr("normal", m, seed=99, ctr_base=shard.counter_base(r))[0]
        ve = oracle.fill_ctr("exp", m, seed=99, ctr_base=shard.counter_base(r))[0]
        want_n = [a + int((np.abs(vn) > t).sum()) for a, t in zip(want_n, scale.C5_THRESH)]
        want_e += int((ve > 2.0).sum())
        allv.append(oracle.fill_ctr("normal", m, seed=scale.C3_SEED,
                                    ctr_base=shard.counter_base(r))[0])
    rep5 = res[0][1]
    assert [row["count"] for row in rep5["normal_abs_tails"]] == want_n
    assert rep5["exp_beyond_X1"]["count"] == want_e > 0
    assert rep5["passed"]
    allv = np.concatenate(allv)
    rep3 = res[0][2]
    assert rep3 == res[1][2]
    assert rep3["n_total"] == total
    assert rep3["mean"] == pytest.approx(float(allv.mean()), rel=1e-9, abs=1e-12)
    assert rep3["passed"]
