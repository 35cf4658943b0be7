import faulthandler, sys, time
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, '.')
import torch, numpy as np
import paper_1403_6870_b200 as zf
dev = torch.device('cuda', 0)
print('start', flush=True)
s = zf.ExpSampler(source=zf.UniformSource.replay([123456789 << 8]), device=dev)
print('sampler ok', flush=True)
t = time.time(); print(s.sample(), time.time() - t, flush=True)
s = zf.ExpSampler(source=zf.UniformSource(7), device=dev)
t = time.time(); print(s.fill(5), time.time() - t, flush=True)
