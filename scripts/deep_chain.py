"""Full-depth K3S chain (128 linears, private output per layer): first
non-finite layer and the per-layer max |y|, per width.
    python scripts/deep_chain.py [B] [widths...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
widths = [int(a) for a in sys.argv[2:]] or [2, 4]
st = LinearStack(LLAMA31_8B, batch=B, n_layers=32)
for r in widths:
    g = torch.Generator(device="cuda").manual_seed(r)
    x0 = torch.randn(B, 4096, device="cuda", generator=g).to(torch.bfloat16)
    layers, X = [], x0
    for _, _, pt in st.layers:
        Y = torch.zeros((B, pt.N), dtype=torch.bfloat16, device="cuda")
        layers.append((pt, X[:, :pt.K], Y))
        X = Y
    prog = mq.StackProgram(layers, r, B)
    prog.run()
    torch.cuda.synchronize()
    bad = [i for i, (_, _, Y) in enumerate(layers) if not torch.isfinite(Y.float()).all()]
    mx = [float(Y.float().abs().max()) for _, _, Y in layers]
    # the same chain through the per-layer K3 path
    mx3 = []
    Xk = x0
    for pt, _, _ in layers:
        Yk = pt.gemv(Xk[:, :pt.K].contiguous(), r)
        mx3.append(float(Yk.float().abs().max()))
        Xk = Yk
    torch.cuda.synchronize()
    print("r=%d first non-finite layer: %s; max|y| K3S %s" % (r, bad[:5], ["%.3g" % v for v in mx[::8]]))
    print("       per-layer K3 max|y| %s" % (["%.3g" % v for v in mx3[::8]]))
