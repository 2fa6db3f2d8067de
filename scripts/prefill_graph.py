"""K4 prefill sweep timed as CUDA graphs (bench.py's prefill_leg):
    python scripts/prefill_graph.py [batches] [bits]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_03537_b200 as mq  # noqa: E402


class _NoClock:
    def active(self, on):
        pass


batches = tuple(int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "64,256,1024").split(","))
bits = tuple(int(b) for b in (sys.argv[2] if len(sys.argv) > 2 else "4").split(","))
out = bench.prefill_leg(torch, mq, _NoClock(), batches=batches, bits=bits)
for k, v in out["per_layer"].items():
    print("%-18s %8.1f us %6.0f TF/s frac %.3f dense %7.1f us vs_dense %.2f" % (
        k, v["us"], v["tflops"], v["frac"], v["dense_bf16_us"], v["vs_dense"]))
for k, v in out["block"].items():
    print("block %-10s %8.1f us %6.0f TF/s frac %.3f vs_dense %.2f" % (k, v["us"], v["tflops"], v["frac"], v["vs_dense"]))
