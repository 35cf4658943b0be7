"""Oracle-mode (sequential xoshiro256++ stream) fill timing, for launch lists.

    python tools/oracle_prof.py [log2 n] [reps] [exp|normal]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 26)
reps = int(sys.argv[2] if len(sys.argv) > 2 else 5)
dist = sys.argv[3] if len(sys.argv) > 3 else "exp"
dev = torch.device("cuda", 0)
cls = zf.ExpSampler if dist == "exp" else zf.NormalSampler
out = torch.empty(n, dtype=torch.float64, device=dev)
s = cls(source=zf.UniformSource(42), device=dev)
s.fill(out)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(reps):
    s.fill(out)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / reps
print(f"oracle mode {dist} n=2^{n.bit_length()-1}: {dt*1e3:.3f} ms/fill, {n/dt/1e9:.2f} G samples/s")
