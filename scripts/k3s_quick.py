"""K3S ms/step and HBM roofline fraction per width (Llama-3.1-8B fused linear
stack, 32 blocks): python scripts/k3s_quick.py [B] [widths...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
widths = [int(a) for a in sys.argv[2:]] or [2, 3, 4, 6, 8]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6525.9
st = LinearStack(LLAMA31_8B, batch=B)
for r in widths:
    st.capture(r, stack_kernel=True)
    for _ in range(5):
        st.step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    e0.record(st.stream)
    for _ in range(n):
        st.step()
    e1.record(st.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    gb = st.step_bytes(st.config) / 1e9
    print("r=%d B=%d %.3f ms/step %.0f tok/s %.0f GB/s frac %.3f" % (r, B, ms, B * 1e3 / ms, gb / ms * 1e3,
                                                                   gb / ms * 1e3 / peak), flush=True)
