"""Host-destination paths for e2e: D2H copy bandwidth vs the kernel writing
straight into pinned host memory (UVA, zero-copy).

    python tools/e2e_probe.py [log2 n]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402
from paper_1403_6870_b200 import _lib  # noqa: E402

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
dev = torch.device("cuda", 0)
host = torch.empty(n, dtype=torch.float64).pin_memory()
dbuf = torch.empty(n, dtype=torch.float64, device=dev)


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


d2h = wall(lambda: host.copy_(dbuf, non_blocking=True))
print(f"raw D2H copy: {8 * n / d2h / 1e9:.1f} GB/s")
s = zf.NormalSampler(source=zf.UniformSource.counter(1), device=dev)
api = wall(lambda: s.fill(host))
print(f"NormalSampler.fill(pinned host): {n / api / 1e9:.2f} G samples/s ({8 * n / api / 1e9:.1f} GB/s)")
lib = _lib.lib()


def direct():
    _lib.check(lib.zf_fill(s._dev_tables.handle, _lib.NORMAL, _lib.F64, 1, 0, host.data_ptr(), n,
                           None, _lib.stream_handle(dev)))
zc = wall(direct)
print(f"kernel writing pinned host memory directly: {n / zc / 1e9:.2f} G samples/s "
      f"({8 * n / zc / 1e9:.1f} GB/s)")
ref = s.__class__(source=zf.UniformSource.counter(1), device=dev).fill(n).cpu()
print("bit-identical:", torch.equal(ref.view(torch.int64), host.view(torch.int64)))
