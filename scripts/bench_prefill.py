"""K4 prefill sweep (BASELINE config C4): Qwen3-14B linear shapes, tokens
B in {64..1024}, r in {4, 8}; TFLOP/s vs the measured bf16 peak and vs a dense
bf16 cuBLAS GEMM of the same shape.

    python scripts/bench_prefill.py [--reps 20] [--bits 4,8] [--batches 64,128,256,512,1024]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200.model import QWEN3_14B, tp_layer_dims  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--bits", default="4,8")
    ap.add_argument("--batches", default="64,128,256,512,1024")
    ap.add_argument("--copies", type=int, default=3, help="weight replicas rotated per rep (L2-cold)")
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    tf_peak = float(peaks.get("bf16_tflops", 1631.2))
    bits = [int(b) for b in args.bits.split(",")]
    batches = [int(b) for b in args.batches.split(",")]
    out = []
    for kind in ("qkv", "o", "gate_up", "down"):
        N, K = tp_layer_dims(QWEN3_14B, kind, 1)
        pts = [mq.PlaneTensor.random_parent(N, K, seed=i) for i in range(args.copies)]
        Wd = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        for B in batches:
            X = torch.randn(B, K, device="cuda").to(torch.bfloat16)
            Y = torch.empty(B, N, device="cuda", dtype=torch.bfloat16)
            flops = 2.0 * B * N * K
            dense = timed(lambda: torch.matmul(X, Wd.t(), out=Y), args.reps)
            for r in bits:
                it = [0]

                def run():
                    pts[it[0] % len(pts)].gemm(X, r, out=Y)
                    it[0] += 1
                t = timed(run, args.reps)
                rec = {"kind": kind, "N": N, "K": K, "B": B, "bits": r, "us": t * 1e6,
                       "tflops": flops / t / 1e12, "frac_bf16_peak": flops / t / 1e12 / tf_peak,
                       "dense_bf16_us": dense * 1e6, "vs_dense": dense / t,
                       "weight_GBps": N * K * (r + 1 if r < 8 else 8) / 8 / t / 1e9}
                out.append(rec)
                print(json.dumps(rec), flush=True)
        del pts
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
