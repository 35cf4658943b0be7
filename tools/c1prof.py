import sys, time
sys.path.insert(0, ".")
import torch
import paper_1403_6870_b200 as zf
dev = torch.device("cuda", 0)
out = torch.empty(1_000_000, dtype=torch.float64, device=dev)
for i in range(3):
    s = zf.ExpSampler(source=zf.UniformSource(42), device=dev)
    s.fill(out)
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(20):
    s = zf.ExpSampler(source=zf.UniformSource(42), device=dev)
    s.fill(out)
torch.cuda.synchronize()
print("wall per fill ms", (time.perf_counter() - t) / 20 * 1e3)
