import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2602_03537_b200 import model as m
from tests.test_gpu_stack import _step
os.environ["MQ_STACK_PAIR"] = "1"
for nl in (1, 2):
    stack = m.LinearStack(m.LLAMA31_8B, batch=3, n_layers=nl)
    x0 = torch.randn(3, 4096, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)).to(torch.bfloat16)
    stack.capture(4, stack_kernel=True)
    want, wb = _step(stack, x0)
    saved = list(stack.layers)
    stack.layers = [(n, k, pt.materialize_child(4)) for n, k, pt in saved]
    stack.capture(4, stack_kernel=True)
    got, gb = _step(stack, x0)
    for k in wb:
        d = (gb[k].float() - wb[k].float()).abs()
        nz = (d > 0).nonzero()
        print(nl, k, tuple(wb[k].shape), "ndiff", nz.shape[0], "maxdiff", float(d.max()),
              "cols", (int(nz[:, 1].min()), int(nz[:, 1].max())) if nz.shape[0] else None,
              "rows", sorted(set(nz[:, 0].tolist())) if nz.shape[0] else None)
