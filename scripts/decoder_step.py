"""A few eager decode steps of the Llama-3.1-8B decoder (B = 1, r = 4): a target for an
ncu launch list (per-kernel durations of the full-model step)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200.llama import LlamaDecoder  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dec = LlamaDecoder(batch=1, bits=4, vocab=1024, n_layers=n)
for _ in range(3):
    with torch.cuda.stream(dec.stream):
        dec._forward()
dec.stream.synchronize()
print("ok")
