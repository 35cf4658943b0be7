"""Race hunt by repetition (compute-sanitizer is closed on this pool): the same
launch repeated many times back to back -- hot, power-capped, with whatever
warp interleavings the run produces -- must give the same bits every time.
The first output of each case is the one the whole-output parity tests compare
with the oracle; every later one is compared with it on the device.

    python tools/soak_determinism.py [reps] > gpurun_out/r02d_soak.jsonl
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
dev = torch.device("cuda", 0)


def same(a, b):
    return bool(torch.equal(a.view(torch.int64), b.view(torch.int64)))


def case(name, n, make, dtype=torch.float64, reps=reps):
    ref = torch.empty(n, dtype=dtype, device=dev)
    out = torch.empty(n, dtype=dtype, device=dev)
    make(ref)
    bad = 0
    t = time.time()
    for _ in range(reps):
        out.fill_(float("nan"))
        make(out)
        iv = torch.int64 if dtype == torch.float64 else torch.int32
        bad += 0 if bool(torch.equal(out.view(iv), ref.view(iv))) else 1
    torch.cuda.synchronize()
    print(json.dumps({"case": name, "n": n, "launches": reps, "mismatching_launches": bad,
                      "samples": n * reps, "seconds": round(time.time() - t, 1)}), flush=True)
    del ref, out
    torch.cuda.empty_cache()


def prod(cls, seed, base=0):
    return lambda dst: cls(source=zf.UniformSource.counter(seed, base), device=dev).fill(dst)


def orac(cls, seed):
    return lambda dst: cls(source=zf.UniformSource(seed), device=dev).fill(dst)


case("production normal f64 2^32 (config 3)", 1 << 32, prod(zf.NormalSampler, 7))
case("production exp f64 2^32", 1 << 32, prod(zf.ExpSampler, 7, 1 << 40))
case("production normal f32 2^30", 1 << 30, prod(zf.NormalSampler, 7), torch.float32)
case("production normal f64 2^24 + 77 (one wave)", (1 << 24) + 77, prod(zf.NormalSampler, 3),
     reps=reps * 10)
reqs = [("exp" if i % 2 else "normal", 8192, i) for i in range(4096)]
plan = zf.BatchPlan([r[0] for r in reqs], [r[1] for r in reqs], [r[2] for r in reqs])
case("config 4 batch (4096 x 8192)", plan.total, lambda dst: plan.fill(out=dst, device=dev),
     reps=reps * 10)
case("oracle mode exp 2^26 (xoshiro256++ seed 42)", 1 << 26, orac(zf.ExpSampler, 42))
case("oracle mode normal 2^20 (xoshiro256++ seed 42)", 1 << 20, orac(zf.NormalSampler, 42),
     reps=reps * 5)
