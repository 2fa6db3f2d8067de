"""Run one GEMV shape a few times (for ncu): python scripts/prof_one.py N K r B [reps]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402

N, K, r, B = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
pts = [mq.PlaneTensor.random_parent(N, K, seed=i) for i in range(reps)]
X = torch.randn(B, K, device="cuda").to(torch.bfloat16)
for pt in pts:
    pt.gemv(X, r)
torch.cuda.synchronize()
print("done")
