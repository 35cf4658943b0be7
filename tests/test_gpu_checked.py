"""Production fills, batches and fused statistics through a ZF_CHECKS=1 build
of the library: device-side checks on every queue slot (inside the queue),
round-scratch index (inside the warp's 32 records), store (inside the
output) and on the staged pack (complete before a round reads it).  A failed
check records its source line, which the library reports back; every value is
also compared with the CPU oracle.  compute-sanitizer is closed on the GPU
pool, so these checks are the race/bounds evidence for the shared-memory
queue, the cooperative round scratch and the split (TMA) table staging."""
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]

_SCRIPT = r"""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1403_6870_b200 as zf
from paper_1403_6870_b200 import _lib, quality
from oracle import oracle
L = _lib.lib()
lines = []
def flag():
    for tag in ("fill", "stats"):
        v = getattr(L, "zf_debug_check_line_" + tag)()
        if v:
            lines.append((tag, v))
bad = []
for dist, cls in (("exp", zf.ExpSampler), ("normal", zf.NormalSampler)):
    for n, base in ((1, 0), (513, 0), (4096, 0), (100003, 7), (1 << 22, 1 << 40), (3 << 20, 5)):
        got = cls(source=zf.UniformSource.counter(1234, base), device="cuda").fill(n).cpu().numpy()
        want = oracle.fill_ctr(dist, n, seed=1234, ctr_base=base)[0]
        if not np.array_equal(got.view(np.uint64), want.view(np.uint64)):
            bad.append((dist, n, base))
        x32 = torch.empty(n, dtype=torch.float32, device="cuda")
        cls(source=zf.UniformSource.counter(1234, base), device="cuda").fill(x32)
        if not np.array_equal(x32.cpu().numpy(), want.astype(np.float32)):
            bad.append((dist, n, base, "f32"))
        flag()
    s = cls(source=zf.UniformSource.counter(9), device="cuda")
    s.fill_counted(1 << 20)
    quality.device_sums(cls(source=zf.UniformSource.counter(3), device="cuda"), 1 << 24,
                        hist=(-6.0, 6.0, 64), thresholds=(2.0, 5.0), abs_thresh=True)
    quality.device_sums(cls(source=zf.UniformSource.counter(3), device="cuda"), 1 << 24,
                        moments=0, thresholds=(9.0,))
    cls(source=zf.UniformSource.counter(3), device="cuda").aggregate(1 << 22)
    flag()
reqs = [("exp" if i % 2 else "normal", 8192 if i % 3 else 777 + i, i) for i in range(300)]
zf.fill_batch(reqs, device="cuda")
torch.cuda.synchronize()
flag()
print("BAD", bad)
print("LINES", lines)
"""


def test_checked_build_fills_and_statistics(cuda):
    lib = ROOT / "build" / "variants" / "checked.so"
    if not lib.exists():
        from paper_1403_6870_b200 import _build
        lib = _build.build_variant("checked", ["ZF_CHECKS=1"])
    env = dict(os.environ, ZF_LIB=str(lib))
    res = subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT)], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=1200)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "BAD []" in res.stdout, res.stdout
    assert "LINES []" in res.stdout, res.stdout
