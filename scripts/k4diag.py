import sys, torch
sys.path.insert(0, '.')
import paper_2602_03537_b200 as mq
n, k, B, r = map(int, sys.argv[1:5])
pt = mq.PlaneTensor.random_parent(n, k, seed=n)
X = torch.randn(B, k, device="cuda").to(torch.bfloat16)
got = pt.gemm(X, r, out_dtype=torch.float32)
torch.cuda.synchronize()
want = X.float() @ pt.decode(r).T
print(n, k, B, r, "err", float((got - want).abs().max() / want.abs().max()))
