"""GEMV tuning sweep (run on the GPU box): per layer shape / bit-width /
launch configuration, time back-to-back launches over distinct (L2-cold)
parents with CUDA events.  Configs are forced through the MQ_GEMV_* env
overrides read by libmatq at launch."""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200.device import algorithmic_bytes  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
COPIES = int(os.environ.get("COPIES", "8"))


def time_cfg(pts, X, out, r, reps=5):
    for pt in pts:
        pt.gemv(X, r, out=out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for pt in pts:
            pt.gemv(X, r, out=out)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / len(pts))
    return best


def main():
    bits = [int(b) for b in os.environ.get("BITS", "2,4,8").split(",")]
    batches = [int(b) for b in os.environ.get("BATCH", "1").split(",")]
    warps = os.environ.get("WARPS", "8,16").split(",")
    stages = os.environ.get("STAGES", "2,3,4,6").split(",")
    splits = os.environ.get("SPLITS", "0").split(",")
    shapes = os.environ.get("SHAPES", "qkv,o,gate_up,down").split(",")
    debugs = os.environ.get("DEBUGS", "0").split(",")
    streams = os.environ.get("STREAMS", "-1").split(",")
    res = []
    for name in shapes:
        N, K = SHAPES[name]
        pts = [mq.PlaneTensor.random_parent(N, K, seed=i) for i in range(COPIES)]
        for B in batches:
            X = torch.randn(B, K, device="cuda").to(torch.bfloat16)
            out = torch.empty(B, N, device="cuda", dtype=torch.bfloat16)
            mq.reserve_workspace(max(pt.workspace_bytes(B) for pt in pts) * 64 + (1 << 22))
            for r, w, d, s, dbg, sk in itertools.product(bits, warps, stages, splits, debugs, streams):
                os.environ["MQ_GEMV_WARPS"], os.environ["MQ_GEMV_STAGES"] = w, d
                os.environ["MQ_GEMV_SPLIT"], os.environ["MQ_GEMV_DEBUG"] = s, dbg
                os.environ["MQ_GEMV_STREAM"] = sk
                us = time_cfg(pts, X, out, r)
                gb = algorithmic_bytes(N, K, B, r, pts[0].planes_read(r)) / (us * 1e-6) / 1e9
                rec = {"layer": name, "N": N, "K": K, "B": B, "r": r, "warps": int(w), "stages": int(d),
                       "split": int(s), "debug": int(dbg), "stream": int(sk), "us": round(us, 2), "GBps": round(gb, 1)}
                res.append(rec)
                print(json.dumps(rec), flush=True)
        del pts
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/sweep.json", "w") as f:
        json.dump(res, f)


if __name__ == "__main__":
    main()
