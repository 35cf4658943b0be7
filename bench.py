#!/usr/bin/env python
"""Benchmark: fp64 N(0,1) / Exponential(1) samples/s on B200, % of HBM write roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json config 3, the configuration the metric is quoted on):
N(0,1) fp64, n = 2^32 samples per GPU per step, seed 7, production counter
stream, GPU g at counter g*2^40 (weak scaling, no collective on the hot path;
the only collective is a SUM allreduce of the validation statistics).  One
step = one `NormalSampler.fill(out)` = one kernel launch writing 32 GiB (far
larger than the 126 MB L2, so no flush is needed between steps).  The
headline leg runs first, on a GPU that has been idle, before the other legs:
exponential fills and generate-and-sum at the same n, the config-2
validation (2^28, seed 1234), the config-5 tail-stress leg (2^36 draws per
distribution over all ranks, generate-and-count), e2e legs and the CPU
baseline.

Roofline: algorithmic bytes = 8 B per fp64 sample written, 0 B read; achieved
GB/s = 8 n / (CUDA-event kernel time) against MEASURED_PEAKS.json hbm_gbs (a
copy), and against a write-only peak measured live on the same GPU.

e2e: the same metric through the public API into HOST memory: pinned host
tensor (device generation + D2H inside the timed region, every step), and a
pageable numpy array (the reference's own `fill(np.empty(n))` usage).

--impl reference: the reference's algorithm on this box's host cores (the CPU
oracle port of zigfast's fill_normal, oracle/zf_oracle.c: xoshiro256++ per
thread, sharded over all host threads with the reference's derive_seed scheme,
quality.py:121-126) on the same n and seed, into one n-sample host array as
the reference's `fill(np.empty(n))` does.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "samples/sec (fp64 normal & exponential) at 1/2/4/8 B200; % of HBM write roofline"
UNIT = "samples/s"
N_DEFAULT = 1 << 32          # config 3: 2^32 per GPU
SEED = 7                     # config 3
C2_N, C2_SEED = 1 << 28, 1234
C5_TOTAL = 1 << 36           # config 5: 2^36 draws per distribution over all ranks
E2E_N = 1 << 28              # bounded e2e sample per rank per step
CPU_CHUNK = 1 << 20          # per-thread reused buffer of the CPU arms
WORKLOAD = ("C3: N(0,1) fp64, n=2^32 per GPU per step, seed 7, counter-based substreams "
            "(GPU g at counter g*2^40)")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--n-per-gpu", "--n", dest="n", type=int, default=N_DEFAULT)
    p.add_argument("--seed", type=int, default=SEED)
    p.add_argument("--cpu-seconds", type=float, default=10.0,
                   help="target duration of the CPU baseline sample")
    p.add_argument("--c5-total", type=int, default=C5_TOTAL)
    p.add_argument("--e2e-n", type=int, default=E2E_N)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-extra", action="store_true",
                   help="headline leg only (no exp / aggregate / C2 / C5 legs)")
    return p.parse_args()


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    OTHER = [("nvmlClocksEventReasonApplicationsClocksSetting", "applications_clocks_setting"),
             ("nvmlClocksEventReasonHwPowerBrakeSlowdown", "hw_power_brake_slowdown"),
             ("nvmlClocksEventReasonSyncBoost", "sync_boost"),
             ("nvmlClocksEventReasonDisplayClockSetting", "display_clock_setting"),
             ("nvmlClocksEventReasonGpuIdle", "gpu_idle")]

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self.temps = []
        self._ready = threading.Event()
        self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _init_nvml(self):
        try:  # in-process NVML: ~microseconds per sample, so short regions get many
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            # every other reason bit too (applications clocks, power brake, sync
            # boost, display, idle), so a low clock always shows its cause
            bits += [getattr(N, a) for a, _ in self.OTHER if hasattr(N, a)]
            self._nvml = (N, h, bits, N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    @staticmethod
    def _instant_power(N, h):
        # instantaneous board power where the driver offers it (the plain
        # power reading is a ~1 s average that lags a 0.15 s timed region)
        try:
            v = N.nvmlDeviceGetFieldValues(h, [N.NVML_FI_DEV_POWER_INSTANT])[0]
            if v.nvmlReturn == 0:
                return v.value.uiVal / 1000.0
        except Exception:
            pass
        return N.nvmlDeviceGetPowerUsage(h) / 1000.0

    def _sample_nvml(self):
        N, h, bits, mx = self._nvml
        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
        pw = self._instant_power(N, h)
        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        try:
            self.temps.append(N.nvmlDeviceGetTemperature(h, N.NVML_TEMPERATURE_GPU))
        except Exception:
            pass
        self.rows.append([str(self.index), str(sm), str(mx), f"{pw:.1f}"] +
                         ["Active" if r & b else "Not Active" for b in bits])

    def _run(self):
        if self._nvml:
            while not self._stop.is_set():
                self._sample_nvml()
                self._ready.set()
                self._stop.wait(0.002)
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.2)

    def __enter__(self):
        self._init_nvml()  # before the timed region starts
        self._t.start()
        self._ready.wait(timeout=10)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if self._nvml:  # one more sample at the end of the region
            self._sample_nvml()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if self._nvml:
            N = self._nvml[0]
            names += [nm for a, nm in self.OTHER if hasattr(N, a)]
        reasons = sorted({names[i] for r in self.rows for i in range(len(names))
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        pw = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None,
                "temp_c_max": max(self.temps) if self.temps else None,
                "samples": len(self.rows)}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _cpu_sample_desc(dist, n, threads, full: bool):
    how = ("into one n-sample output array (the reference's fill(np.empty(n)))" if full else
           f"each thread through a reused {CPU_CHUNK}-sample buffer (no memory for an "
           "n-sample array)")
    return (f"{dist} fp64, n={n} per rep (the config's n per GPU), seed {SEED}, sharded over "
            f"{threads} threads with derive_seed (quality.py:121-126), {how}; "
            f"oracle/zf_oracle.c")


class _CpuFill:
    """The reference's fill on the host cores: n samples into one output array
    (allocated once, first-touched by the first call), or chunked when the
    host cannot hold the array."""

    def __init__(self, dist: str, n: int, seed: int, threads: int):
        import numpy as np
        from oracle import oracle
        self.o, self.dist, self.n, self.seed, self.threads = oracle, dist, n, seed, threads
        try:
            self.out = np.empty(n)
        except MemoryError:
            self.out = None

    @property
    def full(self) -> bool:
        return self.out is not None

    def __call__(self):
        if self.out is not None:
            self.o.fill_sharded(self.dist, self.n, self.seed, threads=self.threads, out=self.out)
        else:
            self.o.fill_sharded_chunked(self.dist, self.n, self.seed, threads=self.threads,
                                        chunk=CPU_CHUNK)


def cpu_baseline(dist: str, n: int, seed: int, seconds: float, threads: int | None = None):
    """The reference algorithm (CPU oracle port) on `threads` host threads on
    the same n and seed as the GPU arm, repeated for about `seconds`."""
    threads = threads or cpu_threads()
    fill = _CpuFill(dist, n, seed, threads)
    fill()  # warm: first touch of the output pages
    times = []
    while not times or (sum(times) < seconds and len(times) < 50):
        t0 = time.perf_counter()
        fill()
        times.append(time.perf_counter() - t0)
    # one host thread, as SURVEY 8(d) asks beside the all-cores figure (the
    # reference's numba fill runs ~0.25 G samples/s per thread in the build
    # container): 2^26 samples into an array of its own, best of 3 after a warm-up
    n1 = min(n, 1 << 26)
    one = _CpuFill(dist, n1, seed, 1)
    one()
    t1 = []
    for _ in range(3):
        t0 = time.perf_counter()
        one()
        t1.append(time.perf_counter() - t0)
    return {"value": n / statistics.median(times), "best": n / min(times), "unit": UNIT,
            "cores": threads, "kind": "port", "reps": len(times),
            "sample": _cpu_sample_desc(dist, n, threads, fill.full), "cpu_model": _cpu_model(),
            "one_thread": {"value": n1 / min(t1), "unit": UNIT, "cores": 1,
                           "sample": f"{dist} fp64, n={n1}, best of 3"}}


def run_reference(args, rank: int):
    """The reference arm: the same workload (n, seed) on the host cores."""
    if rank != 0:
        return
    threads = cpu_threads()
    n = args.n
    fill = _CpuFill("normal", n, args.seed, threads)
    for _ in range(max(1, args.warmup)):
        fill()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fill()
    dt = time.perf_counter() - t0
    value = n * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded)", "impl": "reference",
            "config": {"workload": WORKLOAD, "n_per_gpu": n, "dist": "normal",
                       "seed": args.seed, "cpu_threads": threads},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": _cpu_sample_desc("normal", n, threads, fill.full),
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def timed(fn, steps: int, warmup: int, stream, barrier=None):
    """ms per step of fn() over `steps` calls, CUDA events on `stream`."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        fn()
    t1.record(stream)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / steps


def write_peak(buf, reps: int = 10):
    """Write-only HBM bandwidth on this GPU: torch fill_ (a pure store kernel)."""
    import torch
    for _ in range(3):
        buf.fill_(1.0)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        buf.fill_(1.0)
    t1.record()
    torch.cuda.synchronize()
    return buf.numel() * buf.element_size() * reps / (t0.elapsed_time(t1) * 1e-3) / 1e9


def profile_traffic(n: int):
    """DRAM bytes per launch of the headline kernel from the committed ncu
    capture of this configuration (profiles/), or None."""
    prof = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(prof.read_text())
        rec = d.get("fill_normal_f64", {}).get(str(n))
        if rec:
            return rec["bytes_per_launch"], rec["source"]
    except Exception:
        pass
    return None, None


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:  # lets the driver see the communicator's rank count in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1403_6870_b200 as zf
    from paper_1403_6870_b200 import scale, shard

    # ZF_BENCH_SHARE_DEVICE=1 (tests only, tests/test_gpu_bench_multirank.py):
    # every rank on cuda:0 over gloo, to exercise the N > 1 code path on a
    # one-GPU box -- its numbers are not a scaling measurement
    share = os.environ.get("ZF_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    barrier = dist.barrier if world > 1 else None
    n = args.n
    stream = torch.cuda.current_stream(dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    base = shard.counter_base(rank)

    def sampler(cls, s):
        return cls(source=zf.UniformSource.counter(s, base), device=dev)

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    normal = sampler(zf.NormalSampler, args.seed)
    expo = sampler(zf.ExpSampler, args.seed)
    # every step refills the same counter range: sample k of this rank is
    # global sample g*2^40 + k of seed 7 in every step (fill() of a sampler
    # would advance the stream; the workload is the fixed config-3 range)
    def fill_normal():
        normal.source.state[1] = base
        normal.fill(out)

    def fill_exp():
        expo.source.state[1] = base
        expo.fill(out)

    # -- headline: first, on an idle GPU ------------------------------------------
    fill_normal()
    torch.cuda.synchronize()
    time.sleep(1.0)  # let the power average settle after start-up before the timed leg
    for _ in range(args.warmup):
        fill_normal()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            fill_normal()
        t1.record(stream)
        torch.cuda.synchronize()
    if barrier:
        barrier()
    ms = t0.elapsed_time(t1) / args.steps
    (ms_max,) = max_over_ranks([ms])
    # validation of the last headline step; only these sums cross NCCL
    sums, hist, tails = scale.buffer_stats(out)
    c3 = scale.validate_config3(sums, hist, tails, n, device=dev)

    extra = {}
    if not args.no_extra:
        # each secondary leg starts from the same idle state as the headline
        # (the board's power controller trims long back-to-back runs)
        time.sleep(1.0)
        exp_ms = timed(fill_exp, args.steps, args.warmup, stream, barrier)
        from paper_1403_6870_b200 import quality

        def agg():
            normal.source.state[1] = base
            quality.device_sums(normal, n, moments=1)
        time.sleep(1.0)
        agg_ms = timed(agg, args.steps, args.warmup, stream, barrier)
        # config 2 (validation leg): 2^28, seed 1234
        c2s = zf.NormalSampler(source=zf.UniformSource.counter(C2_SEED, base), device=dev)
        c2o = out[:C2_N]
        c2s.fill(c2o)
        s2, h2, t2 = scale.buffer_stats(c2o)
        c2 = scale.validate_config3(s2, h2, t2, C2_N, device=dev)
        # config 5 (tail stress): total draws per distribution over all ranks
        torch.cuda.synchronize()
        if barrier:
            barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c5 = scale.config5(args.c5_total, rank, world, device=dev)
        e1.record(stream)
        torch.cuda.synchronize()
        exp_ms_max, agg_ms_max, c5_ms_max = max_over_ranks(
            [exp_ms, agg_ms, e0.elapsed_time(e1)])
        extra = {
            "exp_value": n * world / (exp_ms_max * 1e-3), "exp_ms_per_step": exp_ms_max,
            "aggregate": {"value": n * world / (agg_ms_max * 1e-3), "unit": UNIT,
                          "ms_per_step": agg_ms_max, "kernel": "fill_stats_kernel<normal,0>",
                          "note": "generate-and-sum of the same n draws, nothing written "
                                  "(the reference's aggregate / bench loop), timed per "
                                  "quality.device_sums call incl. the partials' merge"},
            "c2_validation": {"workload": "C2: N(0,1) fp64, n=2^28 per GPU, seed 1234", **c2},
            "c5": {"workload": "C5: N(0,1) + Exp(1) fp64, generate-and-count, seed 99",
                   "ms_max_over_ranks": c5_ms_max,
                   "samples_per_s": 2 * args.c5_total / (c5_ms_max * 1e-3), **c5},
        }
    wp = write_peak(out[:1 << 28]) if rank == 0 else None

    # -- e2e through the public API into host memory (rank-local) -------------------
    e2e = None
    if not args.no_e2e:
        m = min(n, args.e2e_n)
        host = torch.empty(m, dtype=torch.float64).pin_memory()
        e2e_s = sampler(zf.NormalSampler, args.seed)
        e2e_s.fill(host[: 1 << 20])
        torch.cuda.synchronize()
        if barrier:
            barrier()
        step_s = []
        t = time.perf_counter()
        for _ in range(args.steps):
            t1 = time.perf_counter()
            e2e_s.fill(host)  # returns when the last chunk's copy has landed
            step_s.append(time.perf_counter() - t1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        arr = np.empty(m)
        e2e_s.fill(arr)  # first call page-locks the array in place (cached while it lives)
        p_steps = max(1, min(args.steps, 5))
        if barrier:
            barrier()
        t = time.perf_counter()
        for _ in range(p_steps):
            e2e_s.fill(arr)
        dtp = time.perf_counter() - t
        # the host link's own D2H rate (a plain pinned copy of the same bytes
        # from HBM), so the e2e number can be read against its bound
        dev_buf = out[:m]
        for _ in range(2):
            host.copy_(dev_buf, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            host.copy_(dev_buf, non_blocking=True)
        torch.cuda.synchronize()
        dtl = (time.perf_counter() - t) / 3
        dt, dtp, dtl = max_over_ranks([dt, dtp, dtl])
        link_gbs = 8 * m / dtl / 1e9
        e2e = {"value": m * world * args.steps / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": 8 * m, "steps": args.steps, "n_per_step": m,
               "step_ms": {"min": 1e3 * min(step_s), "median": 1e3 * float(np.median(step_s)),
                           "max": 1e3 * max(step_s)},
               "note": "NormalSampler.fill(pinned host tensor), every step: device generation + "
                       "D2H copy of the step's 2^28 samples (double-buffered chunks); the input "
                       "is a seed passed by value (no H2D bytes)",
               "pageable": {"value": m * world * p_steps / dtp, "unit": UNIT, "steps": p_steps,
                            "note": "NormalSampler.fill(np.empty(2^28)) repeatedly into the same "
                                    "array, the reference's own usage (exponential.py:45-50): "
                                    "the array is page-locked in place by the first (untimed) "
                                    "call and DMA'd into directly"},
               "link_d2h_gbs_per_gpu": link_gbs,
               "frac_of_link": (m * args.steps / dt) * 8 / 1e9 / link_gbs,
               "link_note": "a pinned cudaMemcpy D2H of the same 8*n bytes on this box: the "
                            "PCIe bound of any host-destination fill (fp64 samples/s <= "
                            "link GB/s / 8 per GPU)"}
        del host

    if rank == 0:
        peak, peak_src = peaks()
        achieved = 8 * n / (ms_max * 1e-3) / 1e9
        traffic, traffic_src = profile_traffic(n)
        line = {
            "metric": METRIC, "value": n * world / (ms_max * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter stream; no dataset)",
            "config": {"workload": WORKLOAD, "n_per_gpu": n, "dist": "normal", "seed": args.seed,
                       "counter_base": "rank * 2^40",
                       "l2": "output 32 GiB per step >> 126 MB L2 (no flush needed)",
                       "parallelism": f"dp{world} (disjoint counter ranges, no hot-path "
                                      "collective)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src,
                         "bytes_per_sample": 8, "write_peak_gbs": wp,
                         "frac_of_write_peak": achieved / wp if wp else None,
                         "kernel": "fill_ctr_kernel<normal,f64>"},
            "validation": {**c3, "allreduce": dist.get_backend() if world > 1 else "none"},
            "clocks": clk.summary(),
            "gpu_launches": args.steps,  # one fill_ctr_kernel launch per timed step
            "e2e": e2e,
            **extra,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline("normal", n, args.seed, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
