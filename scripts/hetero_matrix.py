"""C3 (3.5-bit heterogeneous config over the 224 unfused Llama-3.1-8B linears, or a random
ladder mix over the 128 fused ones): per-layer-r K3S vs the per-layer K3 graph over decode
batches -> LinearStack.stack_kernel_ok.
    python scripts/hetero_matrix.py [batches] [fused]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200.config import budget_config  # noqa: E402
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402


def t_step(stack, n=10):
    for _ in range(3):
        stack.step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stack.stream)
    for _ in range(n):
        stack.step()
    e1.record(stack.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


batches = [int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16").split(",")]
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"
st = LinearStack(LLAMA31_8B, batch=1, fused=fused)
if fused:  # the fused stack's 128 linears: a deterministic mix of the ladder
    import numpy as np

    rng = np.random.default_rng(0)
    cfg = {n: int(rng.choice([2, 3, 4, 6, 8])) for n in st.names}
else:
    cfg = budget_config(3.5, shape=LLAMA31_8B, seed=0, mutations=200).assignment
for B in batches:
    st.set_batch(B)
    row = {}
    for sk in (True, False):
        try:
            st.capture(cfg, stack_kernel=sk)
        except RuntimeError as e:  # the K3S plan may not fit (staging vs ring) at large B
            print("B=%2d K3S plan: %s" % (B, e), flush=True)
            row["K3S"] = float("inf")
            continue
        row["K3S" if sk else "graph"] = t_step(st)
    print("B=%2d hetero3.5  K3S %.3f ms  graph %.3f ms  -> %s" % (B, row["K3S"], row["graph"],
          "K3S" if row["K3S"] < row["graph"] else "graph"), flush=True)
