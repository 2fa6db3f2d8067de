"""Small invocations of every libmatq kernel family for compute-sanitizer
(memcheck / racecheck / synccheck):
    compute-sanitizer --tool racecheck python scripts/sanitize_run.py k3s
Paths: k3s (2-block stack, tiny shapes: stream-K, pair and global split-K
layers, LL hand-off), k3s_llama (one Llama-3.1-8B block), mixed (per-layer r),
k3 (single GEMV, B in {1, 5}), k4 (tcgen05 GEMM), k4tail (whole waves + split tail),
decoder (a tiny Qwen3-style decoder step: K3S segments with fused add+RMSNorm / SiLU
prologues, the decode-attention kernel, glue kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402
from paper_2602_03537_b200.shapes import DecoderShape  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "k3s"
TINY = DecoderShape("tiny", 1024, 4096, 8, 2, 128, 2)
if what in ("k3s", "k3s_llama", "mixed"):
    shape = LLAMA31_8B if what == "k3s_llama" else TINY
    for B in (1, 3):
        st = LinearStack(shape, batch=B, n_layers=1 if what == "k3s_llama" else 2)
        st.x.copy_(torch.randn_like(st.x.float()).to(torch.bfloat16))
        if what == "mixed":
            cfg = {n: (2, 3, 4, 6, 8)[i % 5] for i, n in enumerate(st.names)}
            st.capture(cfg, stack_kernel=True)
        else:
            st.capture(4 if B == 1 else 2, stack_kernel=True)
        for _ in range(2):
            st.program.run(st.stream)
        torch.cuda.synchronize()
        print(what, "B", B, "ok", float(st.x.float().abs().sum()))
elif what == "k3":
    pt = mq.PlaneTensor.random_parent(512, 2048, 128, seed=1)
    for B in (1, 5):
        X = torch.randn(B, 2048, device="cuda").to(torch.bfloat16)
        for r in (2, 4, 8):
            y = pt.gemv(X, r)
        torch.cuda.synchronize()
        print("k3 B", B, "ok", float(y.float().abs().sum()))
elif what == "k4":
    pt = mq.PlaneTensor.random_parent(512, 1024, 128, seed=2)
    X = torch.randn(80, 1024, device="cuda").to(torch.bfloat16)
    for r in (4, 8):
        y = pt.gemm(X, r)
    torch.cuda.synchronize()
    print("k4 ok", float(y.float().abs().sum()))
elif what == "k4tail":
    pt = mq.PlaneTensor.random_parent(2432, 2048, 128, seed=3)
    X = torch.randn(2048, 2048, device="cuda").to(torch.bfloat16)
    y = pt.gemm(X, 4)
    torch.cuda.synchronize()
    print("k4tail ok", float(y.float().abs().sum()))
elif what == "decoder":
    from paper_2602_03537_b200.llama import LlamaDecoder

    shape = DecoderShape("tiny", 512, 1024, 8, 2, 64, 2, qk_norm=True)
    for B in (1, 3):
        dec = LlamaDecoder(shape, batch=B, context=16, bits=4, vocab=1024, linears="k3s")
        dec.tokens.copy_(torch.arange(B, device="cuda") + 1)
        with torch.cuda.stream(dec.stream):
            dec._forward()
        dec.stream.synchronize()
        print("decoder B", B, "ok", float(dec.logits.float().abs().sum()))
