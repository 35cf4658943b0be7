"""One C4 batch (4096 x 8192 mixed requests) for ncu: python tools/prof_c4.py [reps]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1403_6870_b200 as zf  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda", 0)
plan = zf.BatchPlan(["exp" if i % 2 == 0 else "normal" for i in range(4096)], [8192] * 4096,
                    range(4096))
buf = plan.fill(device=dev)
for _ in range(reps):
    plan.fill(buf, device=dev)
torch.cuda.synchronize()
