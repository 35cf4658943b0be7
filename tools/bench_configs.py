"""Measure the non-headline BASELINE.json configs on one B200 (JSON lines).

    python tools/bench_configs.py [c1 c4 c5 f32 ...]

c1   oracle mode: Exponential / N(0,1) fp64, n = 1e6 from UniformSource(42)
     (xoshiro256++, the reference's default stream), parallel resolution of the
     sequential word stream; bit-exactness is asserted by the GPU tests.
c1big  the same pipeline at n = 2^26 (throughput of oracle mode)
c4   4096 requests x 8192 samples, alternating exp/normal, seeds 0..4095:
     one batched launch vs 4096 separate fills
c5   tail stress, config 5 in full on one GPU: N(0,1) and Exp(1), 2^36 each, seed
     99, counts of |x| > 5, 6, 7 and of x > X[1] vs the analytic tail mass
     (5-sigma binomial); generate-and-count, nothing materialised (scale.config5)
f32  fp32 production fills (n = 2^28) for both distributions
trad modified vs traditional ziggurat on the GPU (the paper's Table 1 comparison,
     reference tests/test_acceptance.py criterion 6): fp64 fills n = 2^28 and
     generate-and-sum n = 2^32, production counter streams; plus tail-sample
     agreement of the device log with glibc's over 2^24 draws
fmt  output formats: device '%.17g' text of 2^26 normal draws
     (kernel time, bytes/s of text) vs CPython's f-string join on a 2^20 sample,
     and gen-style end to end (fill + format + D2H) into host memory
agg  generate-and-aggregate (the reference's bench loop):
     sum of n = 2^32 draws with nothing written to HBM (sum-only kernel), and
     the 5-moment validation kernel; kernel time by CUDA events
"""
import json
import math
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402
from paper_1403_6870_b200 import quality  # noqa: E402

dev = torch.device("cuda", 0)


def ev_time(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        fn()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / reps / 1e3  # seconds


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def emit(d):
    print(json.dumps(d), flush=True)


def c1(n=1_000_000, name="c1"):
    for dist, cls in (("exp", zf.ExpSampler), ("normal", zf.NormalSampler)):
        out = torch.empty(n, dtype=torch.float64, device=dev)

        def go():
            s = cls(source=zf.UniformSource(42), device=dev)
            s.fill(out)
        sec = wall(go)
        emit({"config": name, "dist": dist, "n": n, "mode": "oracle (xoshiro256++ seed 42)",
              "seconds_per_fill": sec, "samples_per_s": n / sec,
              "note": "includes device word generation (GF(2) jump-ahead), the parallel "
                      "replay resolution and the host sync that returns words consumed"})


def c4():
    reqs = [("exp" if i % 2 == 0 else "normal", 8192, i) for i in range(4096)]
    total = 4096 * 8192

    t0 = time.perf_counter()
    plan = zf.BatchPlan([d for d, _, _ in reqs], [n for _, n, _ in reqs],
                        [sd for _, _, sd in reqs])
    buf = plan.fill(device=dev)
    torch.cuda.synchronize()
    sec_first = time.perf_counter() - t0
    one_shot = wall(lambda: zf.fill_batch(reqs, device=dev), reps=5)
    sec_b = wall(lambda: plan.fill(buf, device=dev), reps=10)
    sec_k = ev_time(lambda: plan.fill(buf, device=dev), reps=20)
    outs = torch.empty(total, dtype=torch.float64, device=dev)

    def separate():
        for i, (d, n, sd) in enumerate(reqs):
            cls = zf.ExpSampler if d == "exp" else zf.NormalSampler
            cls(source=zf.UniformSource.counter(sd), device=dev).fill(outs[i * n:(i + 1) * n])
    sec_s = wall(separate, reps=1)
    emit({"config": "c4", "requests": 4096, "per_request": 8192,
          "batched_seconds": sec_b, "batched_samples_per_s": total / sec_b,
          "batched_event_seconds": sec_k, "batched_event_samples_per_s": total / sec_k,
          "separate_seconds": sec_s, "separate_samples_per_s": total / sec_s,
          "plan_create_and_first_fill_seconds": sec_first, "one_shot_fill_batch_seconds": one_shot,
          "note": "batched = BatchPlan.fill with the request table resident on the device "
                  "(one zf_batch_fill launch per call); one_shot = zf.fill_batch (table built, "
                  "staged and uploaded every call); separate = 4096 sampler constructions + "
                  "fills through the Python API"})


def c5(total=1 << 36):
    """Config 5 on one GPU (the whole 2^36 per distribution; under torchrun the
    same scale.config5 call splits it over the ranks): generate-and-count in
    the tail-only kernel mode (moments = 0, thresholds above every fast-path
    value), with the full-statistics kernel timed beside it for the record."""
    from paper_1403_6870_b200 import scale
    scale.config5(1 << 24, 0, 1, device=dev)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = scale.config5(total, 0, 1, device=dev)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t
    n = 1 << 33
    s = zf.NormalSampler(source=zf.UniformSource.counter(99), device=dev)
    t = time.perf_counter()
    quality.device_sums(s, n, thresholds=(5.0, 6.0, 7.0), abs_thresh=True)
    torch.cuda.synchronize()
    full = time.perf_counter() - t
    emit({"config": "c5", "n_total_per_dist": total, "seconds": sec,
          "samples_per_s": 2 * total / sec, **rep,
          "full_statistics_kernel_2p33_samples_per_s": n / full,
          "note": "normal |x| > 5, 6, 7 and Exp(1) x > X[1]: tail-only kernel (counts on the "
                  "rare path only) vs the full moments + thresholds kernel on 2^33 normal draws"})


def f32(n=1 << 28):
    for dist, cls in (("exp", zf.ExpSampler), ("normal", zf.NormalSampler)):
        s = cls(source=zf.UniformSource.counter(1234), device=dev)
        out = torch.empty(n, dtype=torch.float32, device=dev)
        sec = ev_time(lambda: s.fill(out))
        emit({"config": "f32", "dist": dist, "n": n, "samples_per_s": n / sec,
              "gbs": 4 * n / sec / 1e9})


def agg(n=1 << 32):
    import ctypes as C
    from paper_1403_6870_b200 import _lib
    for dist, cls in (("exp", zf.ExpSampler), ("normal", zf.NormalSampler)):
        s = cls(source=zf.UniformSource.counter(1234), device=dev)
        row = {"config": "agg", "dist": dist, "n": n}
        for name, moments in (("sum", 1), ("moments5", 5)):
            cfg = quality._cfg(moments=moments)
            partials, counts = quality._buffers(dev, n, cfg)
            lib = _lib.lib()

            def run():
                _lib.check(lib.zf_fill_stats(s._dev_tables.handle, s._dist, 1234, 0, n,
                                             C.byref(cfg), partials.data_ptr(),
                                             counts.data_ptr(), _lib.stream_handle(dev)))
            sec = ev_time(run)
            row[f"{name}_samples_per_s"] = n / sec
        sec = wall(lambda: s.aggregate(n))
        row["aggregate_call_samples_per_s"] = n / sec
        emit(row)
    # validation reductions of an existing 2^28 fp64 buffer (HBM read bound)
    m = 1 << 28
    buf = zf.NormalSampler(source=zf.UniformSource.counter(5), device=dev).fill(m)
    row = {"config": "buffer_stats", "n": m}
    for name, hist in (("moments5", None), ("moments5_hist1024", (-6.0, 6.0, 1024))):
        cfg = quality._cfg(hist=hist)
        partials, counts = quality._buffers(dev, m, cfg)
        lib = _lib.lib()

        def run():
            _lib.check(lib.zf_stats(_lib.F64, buf.data_ptr(), m, C.byref(cfg),
                                    partials.data_ptr(), counts.data_ptr(),
                                    _lib.stream_handle(dev)))
        sec = ev_time(run)
        row[f"{name}_gbs"] = 8 * m / sec / 1e9
    emit(row)


def trad(n=1 << 28, m=1 << 32):
    import ctypes as C
    from paper_1403_6870_b200 import _lib
    sys.path.insert(0, ".")
    from oracle import oracle as orc
    out = torch.empty(n, dtype=torch.float64, device=dev)
    for dist, mod_cls, trad_cls, code in (("exp", zf.ExpSampler, zf.TraditionalExpSampler,
                                           "trad_exp"),
                                          ("normal", zf.NormalSampler,
                                           zf.TraditionalNormalSampler, "trad_normal")):
        row = {"config": "trad", "dist": dist, "n_fill": n, "n_sum": m}
        for algo, cls in (("modified", mod_cls), ("traditional", trad_cls)):
            s = cls(source=zf.UniformSource.counter(1234), device=dev)
            sec = ev_time(lambda: s.fill(out))
            row[f"{algo}_fill_samples_per_s"] = n / sec
            cfg = quality._cfg(moments=1)
            partials, counts = quality._buffers(dev, m, cfg)
            lib = _lib.lib()

            def run():
                _lib.check(lib.zf_fill_stats(s._dev_tables.handle, s._dist, 1234, 0, m,
                                             C.byref(cfg), partials.data_ptr(),
                                             counts.data_ptr(), _lib.stream_handle(dev)))
            row[f"{algo}_sum_samples_per_s"] = m / ev_time(run)
        row["speedup_fill"] = row["modified_fill_samples_per_s"] / row["traditional_fill_samples_per_s"]
        row["speedup_sum"] = row["modified_sum_samples_per_s"] / row["traditional_sum_samples_per_s"]
        k = 1 << 24
        got = trad_cls(source=zf.UniformSource.counter(77), device=dev).fill(k).cpu().numpy()
        want, _, recs = orc.fill_ctr(code, k, seed=77, records=True)
        tail = recs["path"] == 2
        diff = got.view("u8") != want.view("u8")
        row["tail_check"] = {"draws": k, "tail_samples": int(tail.sum()),
                             "mismatches": int(diff.sum()),
                             "non_tail_mismatches": int((diff & ~tail).sum())}
        emit(row)


def fmt(n=1 << 26):
    import ctypes as C
    from paper_1403_6870_b200 import _lib
    from paper_1403_6870_b200.output import format_g17
    s = zf.NormalSampler(source=zf.UniformSource.counter(1), device=dev)
    x = s.fill(n)
    out = torch.empty(24 * n, dtype=torch.uint8, device=dev)
    scratch = torch.zeros(int(_lib.lib().zf_format_scratch_words(n)), dtype=torch.int64,
                          device=dev)
    lib = _lib.lib()

    def run():
        _lib.check(lib.zf_format_g17(x.data_ptr(), n, out.data_ptr(), out.numel(),
                                     scratch.data_ptr(), _lib.stream_handle(dev)))
    sec = ev_time(run)
    nbytes = int(scratch[0].item())
    sample = x[: 1 << 20].cpu().numpy()
    t = time.perf_counter()
    txt = "".join(f"{v:.17g}\n" for v in sample.tolist()).encode()
    cpu = (1 << 20) / (time.perf_counter() - t)
    assert format_g17(x[: 1 << 20]).cpu().numpy().tobytes() == txt
    host = torch.empty(24 * (1 << 24), dtype=torch.uint8).pin_memory()

    def e2e():
        vals = s.fill(1 << 24)
        b = format_g17(vals)
        host[: b.numel()].copy_(b)
    e2e_sec = wall(e2e)
    emit({"config": "fmt", "n": n, "text_bytes": nbytes, "bytes_per_value": nbytes / n,
          "device_values_per_s": n / sec, "device_text_gbs": nbytes / sec / 1e9,
          "cpython_fstring_values_per_s": cpu,
          "gen_e2e_values_per_s": (1 << 24) / e2e_sec})


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c1big", "c4", "c5", "f32"]
    for w in which:
        if w == "c1big":
            c1(1 << 26, "c1big")
        else:
            globals()[w]()
