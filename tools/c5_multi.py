"""BASELINE config 5 across ranks: N(0,1) fp64, n = 2^36 in total, seed 99,
generate-and-count in-kernel (nothing materialised), one rank per GPU.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port 29533 tools/c5_multi.py [log2 total]

Rank r draws its share of the counter stream at counter r * 2^40 (shard.py),
counts |x| > 5, 6, 7 (and Exp(1) draws beyond X[1]) with the fused
statistics kernel, and the only collective is a SUM allreduce of those counts
(NCCL).  Rank 0 prints one JSON line comparing the totals with the analytic
tail mass (binomial 5 sigma) -- the SURVEY 8(d) C5 expectations.
Device time is the max over ranks.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402
from paper_1403_6870_b200 import quality, shard  # noqa: E402

SEED = 99
THRESH = (5.0, 6.0, 7.0)


def main():
    total_log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 36
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    total = 1 << total_log2
    share = total // world + (1 if rank < total % world else 0)
    x1 = float(zf.default_tables("exponential").x[1])
    # warm-up (tables upload, kernel load) outside the timed region
    warm = zf.NormalSampler(source=zf.UniformSource.counter(SEED, shard.counter_base(rank)),
                            device=dev)
    quality.device_sums(warm, 1 << 20, thresholds=THRESH, abs_thresh=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = zf.NormalSampler(source=zf.UniformSource.counter(SEED, shard.counter_base(rank)),
                         device=dev)
    e = zf.ExpSampler(source=zf.UniformSource.counter(SEED, shard.counter_base(rank)), device=dev)
    t0.record()
    _, rn = quality.device_sums(s, share, thresholds=THRESH, abs_thresh=True)
    _, re_ = quality.device_sums(e, share, thresholds=(x1,))
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    counts = shard.allreduce_stats([float(c) for c in rn.thresh_counts] +
                                   [float(re_.thresh_counts[0]), ms if world == 1 else 0.0],
                                   device=dev)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = ms_t.item()
    if rank == 0:
        rows = []
        for th, c in zip(THRESH, counts[:3]):
            ok, mean, sd = quality.binomial_check(int(round(c)), total, math.erfc(th / math.sqrt(2)))
            rows.append({"threshold": th, "count": int(round(c)), "expected": mean, "sd": sd,
                         "within_5sigma": ok})
        ok, mean, sd = quality.binomial_check(int(round(counts[3])), total, math.exp(-x1))
        print(json.dumps({
            "config": "C5: N(0,1) + Exp(1) fp64, generate-and-count, seed 99",
            "n_total_per_dist": total, "n_gpus": world, "ms_max_over_ranks": ms_max,
            "samples_per_s": 2 * total / (ms_max * 1e-3),
            "normal_abs_tails": rows,
            "exp_beyond_X1": {"X1": x1, "count": int(round(counts[3])), "expected": mean,
                              "sd": sd, "within_5sigma": ok},
            "collective": "nccl allreduce of 4 counts" if world > 1 else "none"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
