"""K4 per-CTA phase timeline (MQ_GEMV_TIMING build), 6 launches in one CUDA
graph (PDL), as bench.py's prefill leg times them:
    MQ_LIB_PATH=build/timing/libmatq.so python scripts/gemm_timing.py N K r B"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200 import _lib  # noqa: E402

N, K, r, B = (int(a) for a in sys.argv[1:5])
L = _lib.lib()
L.mq_debug_gemm_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
pts = [mq.PlaneTensor.random_parent(N, K, seed=i) for i in range(3)]
X = torch.randn(B, K, device="cuda").to(torch.bfloat16)
Y = torch.empty(B, N, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for pt in pts:
        pt.gemm(X, r, out=Y, pdl=True, stream=s)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(6):
        pts[i % 3].gemm(X, r, out=Y, pdl=os.environ.get("PDL", "1") == "1", stream=s)
with torch.cuda.stream(s):
    g.replay()
s.synchronize()
buf = np.zeros(64 * 160 * 6, dtype=np.uint64)
assert L.mq_debug_gemm_timestamps(buf.ctypes.data, buf.size) == 0
all_ts = buf.reshape(64, 160, 6).astype(np.float64)
# the graph's 6 launches took the slots after the 3 warm-up launches (and the
# capture, which launches nothing)
slots = [(3 + i) % 64 for i in range(6)]
t00 = min(all_ts[sl][all_ts[sl][:, 0] > 0][:, 0].min() for sl in slots)
names = ["start", "first raw", "first MMA", "last commit", "epilogue", "end"]
for i, sl in enumerate(slots):
    ts = all_ts[sl]
    ts = (ts[ts[:, 0] > 0] - t00) / 1e3
    print("launch %d (%d CTAs): " % (i, len(ts)) + "  ".join(
        "%s %.2f/%.2f" % (n, np.min(ts[:, j]), np.max(ts[:, j])) for j, n in enumerate(names)))
