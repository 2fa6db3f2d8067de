"""mq_attn_decode alone: device time per launch (CUDA graph of 64 launches, PDL chained)
over the context length, Llama-3.1-8B heads (32 q / 8 kv, hd 128), B = 1."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200 import _lib  # noqa: E402

B, nh, nkv, hd = 1, 32, 8, 128
for T in (2, 17, 65, 257, 1025):
    pos = T - 1
    layers = 8
    qkv = torch.randn(B, (nh + 2 * nkv) * hd, device="cuda").to(torch.bfloat16)
    kc = [torch.randn(B, nkv, T, hd, device="cuda").to(torch.bfloat16) for _ in range(layers)]
    vc = [torch.randn(B, nkv, T, hd, device="cuda").to(torch.bfloat16) for _ in range(layers)]
    cos = torch.ones(hd // 2, device="cuda", dtype=torch.bfloat16)
    sin = torch.zeros(hd // 2, device="cuda", dtype=torch.bfloat16)
    kvq = torch.arange(nh, device="cuda", dtype=torch.int32) // (nh // nkv)
    att = torch.empty(B, nh * hd, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()

    def run():
        for i in range(64):
            _lib.call("mq_attn_decode", _lib.ptr(qkv), _lib.ptr(cos), _lib.ptr(sin), None, None, 1e-6,
                      _lib.ptr(kc[i % layers]), _lib.ptr(vc[i % layers]), _lib.ptr(kvq), _lib.ptr(att),
                      B, nh, nkv, hd, T, pos, _lib.stream_ptr(s))
    with torch.cuda.stream(s):
        run()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run()
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(10):
            g.replay()
    e1.record(s)
    e1.synchronize()
    print("T=%5d  %.2f us per launch" % (T, e0.elapsed_time(e1) * 1e3 / 640))
