"""One process, both TP ranks' shards: segment by segment, partials summed by
hand, against the single-GPU stack (debugging tests/test_gpu_tp.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack  # noqa: E402
from tests.conftest import rel_err  # noqa: E402

B = 2
x0 = torch.randn(B, 4096, generator=torch.Generator().manual_seed(5)).to(torch.bfloat16).cuda()
ref = LinearStack(LLAMA31_8B, batch=B, n_layers=1)
ranks = [LinearStack(LLAMA31_8B, batch=B, n_layers=1, tp=2, rank=j, shard_from_full=True) for j in range(2)]
for st in ranks:
    st._all_reduce = lambda t: None  # summed by hand below
for r in (2, 4):
    for sk in (True, False):
        ref.capture(r, stack_kernel=True)
        ref.x.copy_(x0)
        ref.step()
        torch.cuda.synchronize()
        want = {k: v.float().clone() for k, v in ref.bufs.items()}
        want["x"] = ref.x.float().clone()
        # layer by layer through the rank stacks (PlaneTensor.linear), summing partials by hand
        outs = []
        for st in ranks:
            st.x.copy_(x0)
        acc = {}
        for li, kind in enumerate(("qkv", "o", "gate_up", "down")):
            parts = []
            for st in ranks:
                _, _, pt = st.layers[li]
                src = {"qkv": st.x, "o": st.bufs["qkv"][:, :pt.K], "gate_up": st.bufs["o"],
                       "down": st.bufs["gate_up"][:, :pt.K]}[kind]
                y = pt.linear(src, r, out_dtype=torch.float32)
                parts.append(y)
            if kind in ("o", "down"):
                s = parts[0] + parts[1]
                for st in ranks:
                    (st.x if kind == "down" else st.bufs[kind]).copy_(s.to(torch.bfloat16))
                acc[kind] = s
            else:
                for st, y in zip(ranks, parts):
                    st.bufs[kind].copy_(y.to(torch.bfloat16))
        torch.cuda.synchronize()
        print("r=%d manual: o %.4f  x %.4f" % (r, rel_err(acc["o"].cpu().numpy(), want["o"].cpu().numpy()),
                                                 rel_err(acc["down"].cpu().numpy(), want["x"].cpu().numpy())))
        # the TP program path on each rank, all-reduce by hand between segments
        for st in ranks:
            st.capture(r, stack_kernel=sk, graph=False)
            st.x.copy_(x0)
        if sk:
            for seg in range(2):
                for st in ranks:
                    st.programs[seg][0].run(st.stream)
                torch.cuda.synchronize()
                outs = [st.programs[seg][1] for st in ranks]
                s = outs[0].float() + outs[1].float()
                for o in outs:
                    o.copy_(s.to(torch.bfloat16))
                torch.cuda.synchronize()
                if seg == 0:
                    print("  K3S seg0 o vs ref: %.4f" % rel_err(s.cpu().numpy(), want["o"].cpu().numpy()))
            print("  K3S x vs ref: %.4f" % rel_err(ranks[0].x.float().cpu().numpy(), want["x"].cpu().numpy()))
        else:
            for st in ranks:
                st.x.copy_(x0)
            # per-layer K3 path: run layer by layer with hand all-reduce
            for li, kind in enumerate(("qkv", "o", "gate_up", "down")):
                outs = []
                for st in ranks:
                    name, _, pt = st.layers[li]
                    src = {"qkv": st.x, "o": st.bufs["qkv"][:, :pt.K], "gate_up": st.bufs["o"],
                           "down": st.bufs["gate_up"][:, :pt.K]}[kind]
                    out = st.x if kind == "down" else st.bufs[kind]
                    pt.linear(src, r, out=out, pdl=True, stream=st.stream)
                    outs.append(out)
                torch.cuda.synchronize()
                if kind in ("o", "down"):
                    s = outs[0].float() + outs[1].float()
                    for o in outs:
                        o.copy_(s.to(torch.bfloat16))
                    torch.cuda.synchronize()
            print("  K3 x vs ref: %.4f" % rel_err(ranks[0].x.float().cpu().numpy(), want["x"].cpu().numpy()))
