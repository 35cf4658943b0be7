"""Host-side transfer probe (experiment tool): pinned / registered / pageable
D2H rates, host memcpy rates and cudaHostRegister cost on the GPU box."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

GB = 1e9
n = 1 << 28  # doubles (2 GiB)
dev = torch.device("cuda", 0)
src = torch.empty(n, dtype=torch.float64, device=dev).fill_(1.0)
torch.cuda.synchronize()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "torch threads",
      torch.get_num_threads())
os.system("free -g | head -2; lscpu | grep -E 'Model name|Socket|NUMA node|Thread|Core' ")


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


pinned = torch.empty(n, dtype=torch.float64).pin_memory()
dt = t(lambda: pinned.copy_(src, non_blocking=True))
print(f"D2H pinned 2 GiB: {8 * n / dt / GB:.1f} GB/s")

arr = np.empty(n)
arr.fill(0.0)
cart = torch.cuda.cudart()
t0 = time.perf_counter()
rc = cart.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
reg_s = time.perf_counter() - t0
print(f"cudaHostRegister 2 GiB: rc={rc} {reg_s * 1e3:.1f} ms")
host_t = torch.from_numpy(arr)
dt = t(lambda: host_t.copy_(src, non_blocking=True))
print(f"D2H into registered pageable 2 GiB: {8 * n / dt / GB:.1f} GB/s (is_pinned {host_t.is_pinned()})")
t0 = time.perf_counter()
rc = cart.cudaHostUnregister(arr.ctypes.data)
print(f"cudaHostUnregister: rc={rc} {(time.perf_counter() - t0) * 1e3:.1f} ms")
for m in (1 << 20, 1 << 24):  # register cost per size
    a = np.empty(m)
    a.fill(0)
    t0 = time.perf_counter()
    cart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    r = time.perf_counter() - t0
    cart.cudaHostUnregister(a.ctypes.data)
    print(f"cudaHostRegister {a.nbytes >> 20} MiB: {r * 1e3:.2f} ms")

dt = t(lambda: torch.from_numpy(arr).copy_(src))
print(f"D2H pageable (driver path) 2 GiB: {8 * n / dt / GB:.1f} GB/s")
for th in (1, 4, 8, 16, 32):
    torch.set_num_threads(th)
    dt = t(lambda: torch.from_numpy(arr).copy_(pinned))
    print(f"host copy pinned->pageable torch {th} threads: {8 * n / dt / GB:.1f} GB/s")
dt = t(lambda: np.copyto(arr, pinned.numpy()))
print(f"host copy numpy 1 thread: {8 * n / dt / GB:.1f} GB/s")

from oracle import oracle  # noqa: E402
th = len(os.sched_getaffinity(0))
for m in (1 << 28, 1 << 30):
    out = np.empty(m)
    oracle.fill_sharded("normal", m, 7, threads=th, out=out)
    t0 = time.perf_counter()
    oracle.fill_sharded("normal", m, 7, threads=th, out=out)
    dt = time.perf_counter() - t0
    print(f"CPU port full-array fill n=2^{m.bit_length() - 1}: {m / dt / 1e9:.2f} G/s")
t0 = time.perf_counter()
oracle.fill_sharded_chunked("normal", 1 << 30, 7, threads=th)
print(f"CPU port chunked n=2^30: {(1 << 30) / (time.perf_counter() - t0) / 1e9:.2f} G/s")
