"""K3S (the headline persistent decode kernel) against the CPU oracle, layer by
layer, at full model depth and on adversarial activations.

* Full Llama-3.1-8B depth (32 blocks, 128 chained linears) at every ladder
  width: each layer gets its own output buffer, and a sample of its rows is
  recomputed by the oracle (slice_layer -> dense_f32 -> matmul_ref,
  oracle/oracle.py) from the regenerated parent codes and the bf16
  activations the layer actually read.  Bar: bf16 output, max|d|/max|ref|
  <= 1e-2 (reference metric test_matmul.py:19-20).  Outputs
  must be finite -- no skipping.
* Outlier activations (a few channels at 1e3 amid 1e-4 values, all-zero K
  chunks, an all-zero row) through the fp16 staging (r in {4, 8}, B <= 8), the bf16
  two-n-tile path (B = 13, 16) and
  the bf16 zero-point staging (r in {2, 3, 6}).
* The 64-bit step counter: seeded just below 2^32 launches and stepped across
  it (a 32-bit counter would mis-order the layer barriers there).
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

LADDER = (2, 3, 4, 6, 8)


@pytest.fixture(scope="module")
def mq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_03537_b200 as m

    return m


@pytest.fixture(scope="module")
def deep(mq):
    from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack

    return LinearStack(LLAMA31_8B, batch=1, n_layers=32)


def _chain(stack, B, x0):
    """(pt, X, Y) per layer with a private Y per layer: X(l+1) = Y(l)[:, :K(l+1)]."""
    layers, ys = [], []
    X = x0
    for _, _, pt in stack.layers:
        Y = torch.zeros((B, pt.N), dtype=torch.bfloat16, device="cuda")
        layers.append((pt, X[:, :pt.K], Y))
        ys.append(Y)
        X = Y
    return layers, ys


def _oracle_rows(mq, pt, seed_sr, rows, r, X):
    sd, sr, signed = seed_sr if len(seed_sr) == 3 else (*seed_sr, False)
    codes, scales = mq.PlaneTensor.random_parent_codes(pt.N, pt.K, 128, sd, sr, signed)
    idx = torch.as_tensor(rows, device="cuda")
    q = codes[idx].cpu().numpy()
    s = scales[idx].cpu().numpy()
    return O.parent_matmul_ref(q, s, 128, r, X.float().cpu().numpy())


@pytest.mark.parametrize("r", LADDER)
def test_full_depth_every_layer_vs_oracle(mq, deep, r):
    B = 1
    g = torch.Generator(device="cuda").manual_seed(r)
    x0 = torch.randn(B, 4096, device="cuda", generator=g).to(torch.bfloat16)
    layers, ys = _chain(deep, B, x0)
    prog = mq.StackProgram(layers, r, B)
    prog.run()
    torch.cuda.synchronize()
    rng = np.random.default_rng(r)
    worst = 0.0
    for l, ((pt, X, Y), ss) in enumerate(zip(layers, deep.parent_seeds)):
        y = Y.float()
        assert torch.isfinite(y).all(), "layer %d: non-finite output" % l
        rows = np.sort(rng.choice(pt.N, size=48, replace=False))
        want = _oracle_rows(mq, pt, ss, rows, r, X)
        got = y[:, torch.as_tensor(rows, device="cuda")].cpu().numpy()
        e = rel_err(got, want)
        worst = max(worst, e)
        assert e <= 1e-2, "layer %d (%s) r=%d rel err %.3e" % (l, deep.layers[l][0], r, e)
    # a replay is bitwise identical (monotone 64-bit counters, deterministic reductions)
    snap = [Y.clone() for Y in ys]
    prog.run()
    torch.cuda.synchronize()
    for a, b in zip(snap, ys):
        assert torch.equal(a, b)


def _adversarial_x(B, K, kind, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(B, K, device="cuda", generator=g) * 1e-4
    if kind in ("outlier", "both"):
        ch = torch.randint(0, K, (6,), device="cuda", generator=g)
        x[:, ch] = torch.tensor([1e3, -1e3, 7e2, -3e2, 1e3, 5e2], device="cuda")[: ch.numel()]
    if kind in ("zeros", "both"):
        x[:, : min(K, 512)] = 0.0  # whole 256-column steps
        x[:, K // 2: K // 2 + 256] = 0.0
    if B > 1:
        x[-1] = 0.0  # an all-zero row
    return x.to(torch.bfloat16)


@pytest.mark.parametrize("B", [1, 4, 8, 13, 16])
@pytest.mark.parametrize("r", LADDER)
@pytest.mark.parametrize("kind", ["outlier", "zeros", "both"])
def test_adversarial_activations_vs_oracle(mq, r, B, kind):
    """Independent layers (each reads its own crafted X): o-shaped, gate_up-shaped
    (N large) and down-shaped (K = 14336, split-K) parents."""
    shapes = [(4096, 4096), (2048, 4096), (4096, 14336)]
    layers, seeds = [], []
    for i, (N, K) in enumerate(shapes):
        sd, sr = 900 + i, (0.005, 0.02)
        pt = mq.PlaneTensor.random_parent(N, K, 128, sd, sr)
        X = _adversarial_x(B, K, kind, 31 * i + B)
        Y = torch.full((B, N), float("nan"), dtype=torch.bfloat16, device="cuda")
        layers.append((pt, X, Y))
        seeds.append((sd, sr))
    prog = mq.StackProgram(layers, r, B)
    prog.run()
    torch.cuda.synchronize()
    rng = np.random.default_rng(B * 10 + r)
    for (pt, X, Y), ss in zip(layers, seeds):
        y = Y.float()
        assert torch.isfinite(y).all()
        rows = np.sort(rng.choice(pt.N, size=64, replace=False))
        want = _oracle_rows(mq, pt, ss, rows, r, X)
        got = y[:, torch.as_tensor(rows, device="cuda")].cpu().numpy()
        assert rel_err(got, want) <= 1e-2, (pt.N, pt.K, r, B, kind)
        if B > 1:
            assert (y[-1] == 0).all()  # zero activations give exactly zero


def test_step_counter_crosses_2_pow_32(mq):
    from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack

    stack = LinearStack(LLAMA31_8B, batch=2, n_layers=1)
    x0 = torch.randn(2, 4096, device="cuda").to(torch.bfloat16)
    layers, ys = _chain(stack, 2, x0)
    prog = mq.StackProgram(layers, 4, 2)
    prog.run()
    torch.cuda.synchronize()
    want = [y.clone() for y in ys]
    assert prog.launches() == 1
    start = (1 << 32) // 148 - 2  # 148 CTAs: the product crosses 2^32 within 3 steps
    prog.launches(start)
    assert prog.launches() == start
    for i in range(5):
        for y in ys:
            y.zero_()
        prog.run()
        torch.cuda.synchronize()
        for a, b in zip(want, ys):
            assert torch.equal(a, b), "step %d after re-basing" % i
    assert prog.launches() == start + 5
