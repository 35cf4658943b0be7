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
