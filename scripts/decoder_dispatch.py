"""Full-model decode (Llama-3.1-8B shapes, r = 4 unless given): K3S block segments vs per-layer
K3 linears over decode batches -> LlamaDecoder's default `linears` (K3S: B <= 4, the fused add + RMSNorm
prologue stages a whole row).
    python scripts/decoder_dispatch.py [batches] [bits]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200.llama import LlamaDecoder  # noqa: E402

batches = [int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4").split(",")]
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for B in batches:
    row = {}
    for lin in ("k3s", "k3"):
        dec = LlamaDecoder(batch=B, bits=bits, linears=lin)
        dec.tokens.copy_(torch.randint(0, 1000, dec.tokens.shape, device=dec.tokens.device))
        dec.capture()
        for _ in range(3):
            dec.step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dec.stream)
        for _ in range(20):
            dec.step()
        e1.record(dec.stream)
        torch.cuda.synchronize()
        row[lin] = e0.elapsed_time(e1) / 20
        del dec
        torch.cuda.empty_cache()
    print("B=%d r=%d  k3s %.3f ms  k3 %.3f ms  -> %s" % (B, bits, row["k3s"], row["k3"], min(row, key=row.get)),
          flush=True)
