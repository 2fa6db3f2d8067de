"""One K3S decode step of the Llama-3.1-8B linear stack (for ncu):
    python scripts/prof_stack.py [r] [B] [layers]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 32
st = LinearStack(LLAMA31_8B, batch=B, n_layers=nl)
st.capture(r, stack_kernel=True)
for _ in range(3):
    st.program.run(st.stream)
torch.cuda.synchronize()
print("done")
