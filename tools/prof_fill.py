"""Profiling driver: a few production fills of one distribution (for ncu).

    python tools/prof_fill.py [normal|exp] [log2 n] [reps] [f64|f32]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402

dist = sys.argv[1] if len(sys.argv) > 1 else "normal"
n = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 26)
reps = int(sys.argv[3] if len(sys.argv) > 3 else 4)
dt = torch.float32 if (len(sys.argv) > 4 and sys.argv[4] == "f32") else torch.float64
dev = torch.device("cuda", 0)
cls = zf.NormalSampler if dist == "normal" else zf.ExpSampler
s = cls(source=zf.UniformSource.counter(1234), device=dev)
out = torch.empty(n, dtype=dt, device=dev)
for _ in range(reps):
    s.fill(out)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(reps):
    s.fill(out)
t1.record()
torch.cuda.synchronize()
ms = t0.elapsed_time(t1) / reps
print(f"{dist} n=2^{n.bit_length()-1} {dt}: {ms:.4f} ms/launch, {n/ms/1e6:.1f} G samples/s, "
      f"{n*out.element_size()/ms/1e6:.1f} GB/s")
