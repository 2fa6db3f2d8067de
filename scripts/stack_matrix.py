"""K3S vs the per-layer K3 graph over fused / unfused stacks, uniform and
heterogeneous configs (B=1, Llama-3.1-8B, 32 blocks): ms per step."""
import sys

import torch

from paper_2602_03537_b200.config import budget_config
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack


def t_step(stack, n=20):
    for _ in range(3):
        stack.step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stack.stream)
    for _ in range(n):
        stack.step()
    e1.record(stack.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for fused in (True, False):
    st = LinearStack(LLAMA31_8B, batch=B, fused=fused)
    cfgs = [2, 3, 4, 8] if len(sys.argv) < 3 else []
    if fused:
        import numpy as np
        rng = np.random.default_rng(0)
        cfgs.append({n: int(rng.choice([2, 3, 4, 6, 8])) for n in st.names})
    else:
        cfgs.append(budget_config(3.5, shape=LLAMA31_8B, seed=0, mutations=200).assignment)
    for cfg in cfgs:
        row = []
        for sk in (True, False):
            st.capture(cfg, stack_kernel=sk)
            ms = t_step(st)
            gb = st.step_bytes(st.config) / 1e9
            row.append("%s %.3f ms %.0f GB/s" % ("K3S" if sk else "K3g", ms, gb / ms * 1e3))
        print("fused=%d cfg=%s B=%d layers=%d: %s" % (fused, cfg if isinstance(cfg, int) else "C3", B,
                                                     len(st.layers), " | ".join(row)), flush=True)
    del st
    torch.cuda.empty_cache()
