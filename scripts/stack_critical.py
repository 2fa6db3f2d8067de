"""K3S per-layer critical path (MQ_GEMV_TIMING build): for each layer the CTA that
finished last, and how its time split -- wait for the previous layer, staging
(LL wait + conversion), the staging barrier, steps, emit tail, end barrier.
    MQ_LIB_PATH=build/timing/libmatq.so python scripts/stack_critical.py [r] [B]"""
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
L = _lib.lib()
L.mq_debug_stack_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
st = LinearStack(LLAMA31_8B, batch=B)
st.capture(r, stack_kernel=True)
for _ in range(5):
    st.step()
torch.cuda.synchronize()
st.program.run(st.stream)
torch.cuda.synchronize()
buf = np.zeros(256 * 148 * 8 + 256 * 16 * 4, dtype=np.uint64)
assert L.mq_debug_stack_timestamps(buf.ctypes.data, buf.size) == 0
ts = buf[: 256 * 148 * 8].reshape(256, 148, 8).astype(np.float64)[:128]
t0 = ts[0, :, 0].min()
ts = (ts - t0) / 1e3
kinds = ["qkv", "o", "gate_up", "down"]
# events: 0 start, 1 staging done (max warps), 2 after staging barrier, 3 xrow setup,
# 5 last step decoded (max warps), 4 tiles emitted (max warps), 6/7 after end barrier
rows = {k: [] for k in kinds}
prev_end = 0.0
for l in range(128):
    end = ts[l, :, 6]
    c = int(np.argmax(end))
    e = ts[l, c]
    rows[kinds[l % 4]].append([e[0] - prev_end, e[1] - e[0], e[2] - e[1], e[5] - e[2], e[4] - e[5], e[6] - e[4],
                               end.max() - prev_end, np.median(end) - prev_end,
                               (e[3] - e[5]) if e[3] > 0 else np.nan, (e[7] - e[5]) if e[7] > 0 else np.nan])
    prev_end = end.max()
print("step %.1f us; per layer, the last CTA to finish (us):" % prev_end)
print("%-8s %6s %6s %6s %6s %6s %6s | %6s %6s | %6s %6s" % ("", "start", "stage", "sync", "steps", "emit", "endbar",
                                                 "layer", "median", "parts", "remote"))
for k in kinds:
    m = np.nanmean(rows[k], axis=0)
    print("%-8s " % k + " ".join("%6.2f" % v for v in m))
