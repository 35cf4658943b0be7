import sys, time
sys.path.insert(0, '.')
import torch
import paper_1403_6870_b200 as zf
from paper_1403_6870_b200 import _lib
dev = torch.device('cuda', 0)
n = 1 << 26
L = n + n // 8 + 4096
for gen in ("xoshiro256++", "splitmix64"):
    for rep in range(2):
        src = zf.UniformSource(42, generator=gen)
        torch.cuda.synchronize(); t = time.perf_counter()
        w = src.next_block_device(L, dev)
        torch.cuda.synchronize(); print(gen, "words", L, f"{(time.perf_counter()-t)*1e3:.2f} ms", flush=True)
for dist, cls in (("exp", zf.ExpSampler), ("normal", zf.NormalSampler)):
    for rep in range(2):
        s = cls(source=zf.UniformSource.replay(w.cpu().numpy().view("uint64")), device=dev)
        s.source.replay_words_device(dev)
        out = torch.empty(n, dtype=torch.float64, device=dev)
        torch.cuda.synchronize(); t = time.perf_counter()
        s.fill(out)
        torch.cuda.synchronize(); print(dist, "replay fill", n, f"{(time.perf_counter()-t)*1e3:.2f} ms", flush=True)
