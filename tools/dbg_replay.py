"""ZF_DEBUG=1 python tools/dbg_replay.py [normal|exp] [log2 n]: per-stage replay timings."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1403_6870_b200 as zf
dist = sys.argv[1] if len(sys.argv) > 1 else "normal"
n = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 26)
cls = zf.NormalSampler if dist == "normal" else zf.ExpSampler
dev = torch.device('cuda', 0)
out = torch.empty(n, dtype=torch.float64, device=dev)
for _ in range(2):
    cls(source=zf.UniformSource(42), device=dev).fill(out)
    torch.cuda.synchronize()
    print("---", flush=True)
