"""Where the per-block K3S cost goes in the full-model step (Llama-3.1-8B, B = 1, r = 4):
A one K3S launch for all 128 linears (private activation buffers), B the same layers as 32
launches of 4 (no fused prologues), C the decoder's 32 segments (fused add+RMSNorm / SiLU
prologues), D C with the attention kernel between segments.  Device time per step (graph)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200.llama import LlamaDecoder  # noqa: E402
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402


def graph_ms(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


r = int(sys.argv[1]) if len(sys.argv) > 1 else 4
stack = LinearStack(LLAMA31_8B, batch=1, n_layers=32)
x0 = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)
layers, X = [], x0
for _, _, pt in stack.layers:
    Y = torch.zeros((1, pt.N), dtype=torch.bfloat16, device="cuda")
    layers.append((pt, X[:, :pt.K], Y))
    X = Y
one = mq.StackProgram(layers, r, 1)
per = [mq.StackProgram(layers[4 * i:4 * i + 4], r, 1) for i in range(32)]
print("A one launch, 128 layers      %.3f ms" % graph_ms(lambda: one.run(torch.cuda.current_stream())))
print("B 32 launches x 4 layers      %.3f ms" % graph_ms(lambda: [p.run(torch.cuda.current_stream()) for p in per]))
halves = [mq.StackProgram(layers[64 * i:64 * i + 64], r, 1) for i in range(2)]
print("B2 2 launches x 64 layers     %.3f ms" % graph_ms(lambda: [p.run(torch.cuda.current_stream()) for p in halves]))
del one, per, halves, stack, layers
torch.cuda.empty_cache()
dec = LlamaDecoder(batch=1, bits=r, vocab=1024)
dec._build_segments()
from paper_2602_03537_b200 import _lib  # noqa: E402


def segs(keep):
    b, out = dec.buf, []
    for i, blk in enumerate(dec.blocks):
        layers = [(blk["o"].planes, b["att"], b["o"]), (blk["gate_up"].planes, b["o"], b["gu"]),
                  (blk["down"].planes, b["gu"], b["d"])]
        last = i == len(dec.blocks) - 1
        ops = [None, dict(xop=_lib.MQ_XOP_ADD_RMSNORM, res_in=b["x"], res_out=b["xr"] if last else None,
                          norm_w=blk["ln2"], eps=1e-5), dict(xop=_lib.MQ_XOP_SILU_MUL)]
        if not last:
            layers.append((dec.blocks[i + 1]["qkv"].planes, b["d"], b["qkv"]))
            ops.append(dict(xop=_lib.MQ_XOP_ADD_RMSNORM, res_in=None, res_out=b["x"], norm_w=dec.blocks[i + 1]["ln1"],
                            eps=1e-5))
        ops = [o if (o is not None and o["xop"] in keep) else None for o in ops]
        out.append(mq.StackProgram(layers, r, 1, ops=ops if any(ops) else None))
    return out


for name, keep in (("C0 decoder layers, no prologues", ()), ("C1 add+RMSNorm prologues only", (_lib.MQ_XOP_ADD_RMSNORM,)),
                   ("C2 SiLU prologue only", (_lib.MQ_XOP_SILU_MUL,))):
    ps = segs(keep)
    print("%-30s%.3f ms" % (name, graph_ms(lambda: [p.run(torch.cuda.current_stream()) for p in ps])))
    del ps
print("C decoder segments (xops)     %.3f ms" % graph_ms(lambda: [p.run(torch.cuda.current_stream()) for p in dec.segments]))
print("D segments + attention        %.3f ms" % graph_ms(lambda: dec._forward_k3s(parts=("linear", "attn"))))
print("E full step                   %.3f ms" % graph_ms(lambda: dec._forward_k3s()))
