"""Critical path of one decoder block segment (MQ_GEMV_TIMING build): the K3S launch
[o, gate_up (+ add/RMSNorm), down (+ SiLU), next qkv (+ add/RMSNorm)] with and without its
fused prologues.  Per layer, the CTA that finished last: start (after the previous layer's
end), staging, staging barrier, steps, emit, end barrier; plus the layer's median end.
    MQ_LIB_PATH=build/timing/libmatq.so python scripts/segment_critical.py [r]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_03537_b200 as mq  # noqa: E402
from paper_2602_03537_b200 import _lib  # noqa: E402
from paper_2602_03537_b200.llama import LlamaDecoder  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 4
L = _lib.lib()
L.mq_debug_stack_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
dec = LlamaDecoder(batch=1, bits=r, vocab=1024, n_layers=3)
dec.step()
torch.cuda.synchronize()
b, blk, nxt = dec.buf, dec.blocks[1], dec.blocks[2]
layers = [(blk["o"].planes, b["att"], b["o"]), (blk["gate_up"].planes, b["o"], b["gu"]),
          (blk["down"].planes, b["gu"], b["d"]), (nxt["qkv"].planes, b["d"], b["qkv"])]
ops = [None, dict(xop=_lib.MQ_XOP_ADD_RMSNORM, res_in=b["x"], res_out=None, norm_w=blk["ln2"], eps=1e-5),
       dict(xop=_lib.MQ_XOP_SILU_MUL),
       dict(xop=_lib.MQ_XOP_ADD_RMSNORM, res_in=None, res_out=b["xr"], norm_w=nxt["ln1"], eps=1e-5)]
kinds = ["o", "gate_up", "down", "qkv"]
for name, prog in (("no prologues", mq.StackProgram(layers, r, 1)), ("fused prologues", mq.StackProgram(layers, r, 1, ops=ops))):
    for _ in range(5):
        prog.run()
    torch.cuda.synchronize()
    tot, subs = [], []
    for _ in range(5):
        prog.run()
        torch.cuda.synchronize()
        buf = np.zeros(256 * 148 * 8 + 256 * 16 * 4, dtype=np.uint64)
        assert L.mq_debug_stack_timestamps(buf.ctypes.data, buf.size) == 0
        full = buf[: 256 * 148 * 8].reshape(256, 148, 8).astype(np.float64)
        ts = full[:4]
        t0 = ts[0, :, 0].min()
        ts = (ts - t0) / 1e3
        sub = np.where(full[128:132] > 0, (full[128:132] - t0) / 1e3, np.nan)
        subs.append([[np.nanmax(sub[l, :, k]) - ts[l, :, 0].max() if np.isfinite(sub[l, :, k]).any() else np.nan
                      for k in range(6)] + [ts[l, :, 1].max() - ts[l, :, 0].max()] for l in range(4)])
        rows, prev_end = [], 0.0
        for l in range(4):
            end = ts[l, :, 6]
            c = int(np.argmax(end))
            e = ts[l, c]
            rows.append([e[0] - prev_end, e[1] - e[0], e[2] - e[1], e[5] - e[2], e[4] - e[5], e[6] - e[4],
                         end.max() - prev_end, np.median(end) - prev_end, ts[l, :, 0].max() - ts[l, :, 0].min()])
            prev_end = end.max()
        tot.append(rows)
    m = np.median(np.array(tot), axis=0)
    print("== %s: segment %.2f us (kernel start skew %.2f us)" % (name, m[:, 6].sum(), m[0, 8]))
    print("%-8s %6s %6s %6s %6s %6s %6s | %6s %6s" % ("", "start", "stage", "sync", "steps", "emit", "endbar",
                                                     "layer", "median"))
    for k in range(4):
        print("%-8s " % kinds[k] + " ".join("%6.2f" % v for v in m[k, :8]))
    sm = np.nanmedian(np.array(subs), axis=0)
    print("staging sub-phases (latest warp, us after the latest CTA's layer start): delta-arrived, prepass-done, "
          "sync, inv, X-ready, silu-done, staged")
    for k in range(4):
        print("%-8s " % kinds[k] + " ".join("%6.2f" % v for v in sm[k]))
