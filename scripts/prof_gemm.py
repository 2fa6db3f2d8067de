"""Run one K4 shape a few times (for ncu): python scripts/prof_gemm.py N K r B [reps]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402

N, K, r, B = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
pt = mq.PlaneTensor.random_parent(N, K, seed=0)
X = torch.randn(B, K, device="cuda").to(torch.bfloat16)
for _ in range(reps):
    pt.gemm(X, r)
torch.cuda.synchronize()
print("done")
