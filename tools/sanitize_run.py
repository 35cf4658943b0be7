"""Small end-to-end exercise of every kernel family for compute-sanitizer runs."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1403_6870_b200 as zf
from paper_1403_6870_b200 import quality

dev = torch.device("cuda", 0)
for cls in (zf.ExpSampler, zf.NormalSampler):
    s = cls(source=zf.UniformSource.counter(5), device=dev)
    s.fill(100_003)
    s.fill_counted(4097)
    buf = torch.zeros(10_001, dtype=torch.float64, device=dev)
    s.fill(buf[1:])
    s.fill(torch.empty(5000, dtype=torch.float32, device=dev))
    quality.device_sums(s, 50_000, hist=(-6.0, 6.0, 64), thresholds=(1.0,))
    o = cls(source=zf.UniformSource(42), device=dev)
    o.fill_records(20_000)
    r = cls(source=zf.UniformSource.replay([255, 0, 0, 123456789 << 8]), device=dev)
    r.fill(100)
zf.fill_batch([("exp", 1000, 1), ("normal", 8192, 2), ("exp", 3, 3)], device=dev)
# staging-ring reuse and growth, cooperative normal rounds in the batch kernel
zf.fill_batch([("normal", 20_000 + i, 10 + i) for i in range(40)], device=dev)
zf.fill_batch([("exp", 5, 1)], device=dev)
torch.cuda.synchronize()
print("sanitize run ok")
