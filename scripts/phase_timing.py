"""K3 phase timeline from a MQ_GEMV_TIMING build (profiling only):

    MQ_LIB_PATH=build/timing/libmatq.so python scripts/phase_timing.py [B] [r]

Captures, per Llama layer kind, a CUDA graph of 16 same-kind K3 launches
(PDL, as in the decode stack), replays it, and prints per launch the phase
times (median / max over CTAs, us, relative to the earliest CTA entry of
that launch): entry, after griddepcontrol.wait, after X staging, after the
zero-point constants, last unit's fixup start, stream end; plus the gap from
the previous launch's last CTA to this launch's first entry."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200 import _lib  # noqa: E402
from paper_2602_03537_b200.model import LLAMA31_8B, full_layer_dims  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
r = int(sys.argv[2]) if len(sys.argv) > 2 else 4
L = _lib.lib()
L.mq_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.mq_debug_reset.argtypes = []
SLOTS, CTAS, EV = 64, 160, 6
NAMES = ["entry", "wait", "xstage", "zc", "fixup", "end"]
for kind in ("qkv", "o", "gate_up", "down"):
    N, K = full_layer_dims(LLAMA31_8B, kind)
    n = 16
    pts = [mq.PlaneTensor.random_parent(N, K, seed=i) for i in range(n)]
    X = torch.randn(B, K, device="cuda").to(torch.bfloat16)
    Y = torch.empty(B, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    mq.reserve_workspace(max(pt.workspace_bytes(B) for pt in pts), stream=s)
    with torch.cuda.stream(s):
        for pt in pts:
            pt.gemv(X, r, out=Y, pdl=True, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for pt in pts:
            pt.gemv(X, r, out=Y, pdl=True, stream=s)
    for _ in range(3):
        with torch.cuda.stream(s):
            g.replay()
    s.synchronize()
    assert L.mq_debug_reset() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    s.synchronize()
    buf = np.zeros(SLOTS * CTAS * EV, dtype=np.uint64)
    assert L.mq_debug_timestamps(buf.ctypes.data, buf.size) == 0
    ts = buf.reshape(SLOTS, CTAS, EV).astype(np.float64)
    used = [i for i in range(SLOTS) if ts[i, :, 0].max() > 0]
    used.sort(key=lambda i: ts[i, :, 0][ts[i, :, 0] > 0].min())
    print("== %s %dx%d r=%d B=%d: graph of %d launches %.2f us/launch (events)" % (
        kind, N, K, r, B, n, e0.elapsed_time(e1) * 1e3 / n))
    prev_end = None
    for i in used[-6:]:
        t = ts[i]
        act = t[:, 0] > 0
        t0 = t[act, 0].min()
        row = []
        for e in range(EV):
            v = t[act, e]
            v = v[v > 0] - t0
            row.append("%s %5.2f/%5.2f" % (NAMES[e], np.median(v) / 1e3, v.max() / 1e3) if v.size else "%s -" % NAMES[e])
        gap = "" if prev_end is None else " gap_from_prev_end %.2f" % ((t0 - prev_end) / 1e3)
        prev_end = max(t[act, 4].max(), t[act, 0].max())
        print("  ctas %3d | %s%s" % (act.sum(), " | ".join(row), gap))
    del pts
    torch.cuda.empty_cache()
