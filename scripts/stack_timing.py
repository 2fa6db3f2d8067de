"""K3S per-layer phase timeline (MQ_GEMV_TIMING build):
    MQ_LIB_PATH=build/timing/libmatq.so python scripts/stack_timing.py [r] [B] [layers]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200 import _lib  # noqa: E402
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 32
L = _lib.lib()
L.mq_debug_stack_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
st = LinearStack(LLAMA31_8B, batch=B, n_layers=nl)
st.capture(r, stack_kernel=True)
for _ in range(5):
    st.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st.stream)
st.step()
e1.record(st.stream)
torch.cuda.synchronize()
print("step %.1f us (%d layers)" % (e0.elapsed_time(e1) * 1e3, 4 * nl))
buf = np.zeros(256 * 148 * 8 + 256 * 16 * 4, dtype=np.uint64)
assert L.mq_debug_stack_timestamps(buf.ctypes.data, buf.size) == 0
ts = buf[: 256 * 148 * 8].reshape(256, 148, 8).astype(np.float64)[: 4 * nl]
# ev5 is an atomicMax over warps (0 when a CTA had no work for the layer): fall back to ev4
ts[:, :, 5] = np.where(ts[:, :, 5] > 0, ts[:, :, 5], ts[:, :, 4])
t0 = ts[0, :, 0].min()
ts = (ts - t0) / 1e3
kinds = ["qkv", "o", "gate_up", "down"]
# phases (mean over blocks of the per-layer max over CTAs of each event, minus the previous event's max)
names = ["arrive", "released", "staged", "zc", "w0_loop_end", "all_loops", "reduced", "published"]
for k in range(4):
    rows = []
    for l in range(k, 4 * nl, 4):
        mx = ts[l].max(axis=0)
        prev_pub = ts[l - 1, :, 7].max() if l > 0 else mx[0]
        rows.append([mx[1] - prev_pub, mx[2] - mx[1], mx[5] - mx[3], mx[4] - mx[5], mx[6] - mx[4], mx[7] - mx[6]])
    m = np.mean(rows, axis=0)
    print("%-8s " % kinds[k] + "  ".join("%s %.2f" % (n, v) for n, v in zip(
        ["release", "stage", "steps(all warps)", "then w0 done", "barrier", "publish"], m)))
