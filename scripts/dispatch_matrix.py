"""K3S vs the per-layer K3 graph (fused Llama-3.1-8B stack, uniform r) over
decode batches: ms per step -> the LinearStack.stack_kernel_ok table.
    python scripts/dispatch_matrix.py [batches] [widths]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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


batches = [int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8,16").split(",")]
widths = [int(b) for b in (sys.argv[2] if len(sys.argv) > 2 else "2,3,4,6,8").split(",")]
st = LinearStack(LLAMA31_8B, batch=1)
for B in batches:
    st.set_batch(B)
    for r in widths:
        row = {}
        for sk in (True, False):
            st.capture(r, stack_kernel=sk)
            row["K3S" if sk else "graph"] = t_step(st)
        print("B=%2d r=%d  K3S %.3f ms  graph %.3f ms  -> %s" % (B, r, row["K3S"], row["graph"],
              "K3S" if row["K3S"] < row["graph"] else "graph"), flush=True)
