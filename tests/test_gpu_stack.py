"""K3S (one persistent kernel per decode step): every layer's output against
an fp32 torch product of the exactly decoded weights and the activations the
layer actually read (the bf16 tolerance of SURVEY 8(c)); bitwise replay
determinism (the completion counters only grow); agreement with the
per-layer K3 graph; mode C."""

import numpy as np
import pytest
import torch

from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

LADDER = (2, 3, 4, 6, 8)


@pytest.fixture(scope="module")
def model():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.backends.cuda.matmul.allow_tf32 = False
    from paper_2602_03537_b200 import model as m

    return m


def _step(stack, x0):
    stack.x.copy_(x0)
    stack.step()
    torch.cuda.synchronize()
    return stack.x.clone(), {k: v.clone() for k, v in stack.bufs.items()}


def _check_layers(stack, r, x0, y, bufs, tol=1e-2):
    qkv, o, gu, down = (pt for _, _, pt in stack.layers[:4])
    ins = {"qkv": x0, "o": bufs["qkv"][:, :o.K], "gate_up": bufs["o"], "down": bufs["gate_up"][:, :down.K]}
    outs = {"qkv": bufs["qkv"], "o": bufs["o"], "gate_up": bufs["gate_up"], "down": y}
    for kind, pt in zip(("qkv", "o", "gate_up", "down"), (qkv, o, gu, down)):
        want = ins[kind].float() @ pt.decode(r).T
        got = outs[kind].float()
        assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= tol, (kind, r)


@pytest.mark.parametrize("B", [1, 5, 16])
def test_stack_kernel_layers_vs_fp32(model, B):
    stack = model.LinearStack(model.LLAMA31_8B, batch=B, n_layers=1)
    g = torch.Generator(device="cuda").manual_seed(B)
    x0 = torch.randn(B, 4096, device="cuda", generator=g).to(torch.bfloat16)
    for r in LADDER:
        stack.capture(r, stack_kernel=True)
        assert stack.launches_per_step() == 1
        y, bufs = _step(stack, x0)
        assert torch.isfinite(y.float()).all(), r
        _check_layers(stack, r, x0, y, bufs)
        for _ in range(2):  # replays: counters keep growing, results are bitwise stable
            y2, b2 = _step(stack, x0)
            torch.testing.assert_close(y2, y, rtol=0, atol=0)
            for k in bufs:
                torch.testing.assert_close(b2[k], bufs[k], rtol=0, atol=0)
        # the per-layer K3 graph computes the same first layer (other reduction order)
        stack.capture(r, stack_kernel=False)
        _, wb = _step(stack, x0)
        assert rel_err(wb["qkv"].float().cpu().numpy(), bufs["qkv"].float().cpu().numpy()) <= 1e-2


def test_stack_kernel_two_blocks_and_children(model):
    stack = model.LinearStack(model.LLAMA31_8B, batch=3, n_layers=2)
    x0 = torch.randn(3, 4096, device="cuda").to(torch.bfloat16)
    stack.capture(4, stack_kernel=True)
    want, _ = _step(stack, x0)
    assert torch.isfinite(want.float()).all()
    saved = list(stack.layers)
    stack.layers = [(n, k, pt.materialize_child(4)) for n, k, pt in saved]
    stack.capture(4, stack_kernel=True)
    got, _ = _step(stack, x0)
    assert torch.equal(got, want)  # mode C decodes the same codes in the same order
    stack.layers = saved


def test_configs_default_to_stack_kernel(model):
    stack = model.LinearStack(model.LLAMA31_8B, batch=2, n_layers=1)
    stack.capture(3)
    assert stack.program is not None
    cfg = {n: (2 if i % 2 else 4) for i, n in enumerate(stack.names)}
    stack.capture(cfg)  # heterogeneous fused: the per-layer dispatch kernel
    assert stack.program is not None and stack.launches_per_step() == 1
    stack.capture(cfg, stack_kernel=False)  # or the per-layer K3 graph
    assert stack.program is None and stack.launches_per_step() == len(stack.names)
    un = model.LinearStack(model.LLAMA31_8B, batch=2, n_layers=1, fused=False)
    un.capture({n: (2 if i % 2 else 4) for i, n in enumerate(un.names)})  # heterogeneous unfused: K3S too
    assert un.program is not None
    un.capture(3)  # uniform unfused: K3S
    assert un.program is not None


def _check_mixed(stack, cfg, x0, y, bufs, tol=1e-2):
    """One block (4 layers): each layer at its own r against fp32."""
    (nq, _, qkv), (no, _, o), (ng, _, gu), (nd, _, down) = stack.layers[:4]
    ins = {nq: x0, no: bufs["qkv"][:, :o.K], ng: bufs["o"], nd: bufs["gate_up"][:, :down.K]}
    outs = {nq: bufs["qkv"], no: bufs["o"], ng: bufs["gate_up"], nd: y}
    for name, pt in zip((nq, no, ng, nd), (qkv, o, gu, down)):
        got = outs[name].float()
        assert torch.isfinite(got).all(), (name, cfg[name])
        want = ins[name].float() @ pt.decode(cfg[name]).T
        assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= tol, (name, cfg[name])


@pytest.mark.parametrize("B", [1, 4, 12])
def test_stack_kernel_heterogeneous(model, B):
    """Per-layer r inside one persistent kernel: every width of the ladder
    across the layer kinds, each layer against fp32, replays bitwise stable,
    and the same numbers as the per-layer K3 graph within bf16 tolerance."""
    stack = model.LinearStack(model.LLAMA31_8B, batch=B, n_layers=1)
    g = torch.Generator(device="cuda").manual_seed(100 + B)
    x0 = torch.randn(B, 4096, device="cuda", generator=g).to(torch.bfloat16)
    for shift in range(len(LADDER)):
        cfg = {n: LADDER[(i + shift) % len(LADDER)] for i, n in enumerate(stack.names)}
        stack.capture(cfg, stack_kernel=True)
        assert stack.program is not None and stack.launches_per_step() == 1
        y, bufs = _step(stack, x0)
        _check_mixed(stack, cfg, x0, y, bufs)
        y2, b2 = _step(stack, x0)
        torch.testing.assert_close(y2, y, rtol=0, atol=0)
        stack.capture(cfg, stack_kernel=False)
        _, wb = _step(stack, x0)
        assert rel_err(wb["qkv"].float().cpu().numpy(), bufs["qkv"].float().cpu().numpy()) <= 1e-2


@pytest.mark.parametrize("fused", [True, False])
def test_stack_kernel_heterogeneous_multiblock(model, fused):
    """An EvoPress-like random per-layer config over 3 blocks (12 fused / 21
    unfused linears; unfused layers also read outputs older than the previous
    layer's)."""
    stack = model.LinearStack(model.LLAMA31_8B, batch=1, n_layers=3, fused=fused)
    rng = np.random.default_rng(7)
    cfg = {n: int(rng.choice(LADDER)) for n in stack.names}
    x0 = torch.randn(1, 4096, device="cuda").to(torch.bfloat16) * 0.5
    stack.capture(cfg, stack_kernel=True)
    y, _ = _step(stack, x0)
    stack.capture(cfg, stack_kernel=False)
    y_ref, _ = _step(stack, x0)
    assert torch.isfinite(y.float()).all() and torch.isfinite(y_ref.float()).all()
    assert rel_err(y.float().cpu().numpy(), y_ref.float().cpu().numpy()) <= 3e-2


def test_llama_decoder_full_model_step(model):
    """Full-model harness: one captured decode step runs, the projections equal
    their MatLinear (K3) outputs, logits are finite and bit-switching re-captures."""
    from paper_2602_03537_b200.llama import LlamaDecoder

    dec = LlamaDecoder(batch=2, context=64, bits=4, n_layers=2, vocab=4096)
    toks = torch.tensor([3, 7])
    nxt = dec.decode(toks)
    torch.cuda.synchronize()
    assert nxt.shape == (2,) and torch.isfinite(dec.logits.float()).all()
    # eager forward == graph replay
    ref = dec.logits.clone()
    with torch.cuda.stream(dec.stream):
        dec._forward()
    dec.stream.synchronize()
    assert torch.equal(dec.logits, ref)
    dec.set_bits(2)
    dec.decode(toks)
    torch.cuda.synchronize()
    assert not torch.equal(dec.logits, ref)


@pytest.mark.parametrize("B", [1, 9])
def test_stack_kernel_pair_and_global_split_k(model, B, monkeypatch):
    """CTA pairs (clusters of 2, S = 2 reduced through DSMEM) and plain CTAs
    (split-K through the global workspace and tickets) both match fp32 per layer."""
    g = torch.Generator(device="cuda").manual_seed(40 + B)
    x0 = torch.randn(B, 4096, device="cuda", generator=g).to(torch.bfloat16)
    outs = []
    for pair in ("1", "0"):
        monkeypatch.setenv("MQ_STACK_PAIR", pair)
        stack = model.LinearStack(model.LLAMA31_8B, batch=B, n_layers=1)
        for r in (2, 4, 8):
            stack.capture(r, stack_kernel=True)
            y, bufs = _step(stack, x0)
            assert torch.isfinite(y.float()).all(), (pair, r)
            _check_layers(stack, r, x0, y, bufs)
            outs.append(bufs["qkv"])
    for a, b in zip(outs[:3], outs[3:]):
        assert rel_err(a.float().cpu().numpy(), b.float().cpu().numpy()) <= 1e-2


def test_llama_fused_glue_matches_torch_glue(model):
    """The harness's fused glue kernels (residual + RMSNorm, rotary + KV write,
    SiLU gating) against the plain-torch statement of the same decode step."""
    from paper_2602_03537_b200.llama import LlamaDecoder

    outs = {}
    for glue in ("cuda", "torch"):
        dec = LlamaDecoder(batch=3, context=32, bits=4, n_layers=2, vocab=2048, glue=glue)
        dec.tokens.copy_(torch.tensor([5, 9, 100], device="cuda"))
        with torch.cuda.stream(dec.stream):
            dec._forward()
        dec.stream.synchronize()
        outs[glue] = dec.logits.float().clone()
    assert torch.isfinite(outs["cuda"]).all()
    assert rel_err(outs["cuda"].cpu().numpy(), outs["torch"].cpu().numpy()) <= 2e-2


@pytest.mark.parametrize("B", [1, 3])
@pytest.mark.parametrize("r", [2, 4, 8])
def test_stack_gated_output_epilogue(model, B, r):
    """MQ_YOP_SILU_PAIRS: an interleaved gate/up parent (8 gate rows, then their 8 up
    rows, per 16-row tile) writes bf16(bf16(silu(bf16 g)) * bf16 u) as it finishes each
    tile, and the next layer stages it through the LL words: against the same parent run
    as a plain layer, split and gated in torch (the rounding torch's glue applies)."""
    import paper_2602_03537_b200 as mq
    from paper_2602_03537_b200 import _lib
    from paper_2602_03537_b200.llama import LlamaDecoder

    inter, K = 1024, 2048
    perm = LlamaDecoder._glu_rows(inter, "cuda")
    codes, scales = mq.PlaneTensor.random_parent_codes(2 * inter, K, 128, 11, (0.005, 0.02), True)
    gu = mq.PlaneTensor.from_codes(codes[perm].contiguous(), 8, scales[perm].contiguous(), 128)
    down = mq.PlaneTensor.random_parent(512, inter, 128, 12, (0.005, 0.02))
    g = torch.Generator(device="cuda").manual_seed(B + r)
    X = torch.randn(B, K, device="cuda", generator=g).to(torch.bfloat16)
    act = torch.full((B, inter), float("nan"), dtype=torch.bfloat16, device="cuda")
    Y = torch.full((B, 512), float("nan"), dtype=torch.bfloat16, device="cuda")
    prog = mq.StackProgram([(gu, X, act), (down, act, Y)], r, B,
                           ops=[dict(yop=_lib.MQ_YOP_SILU_PAIRS), None])
    prog.run()
    # reference: the same interleaved parent as a plain layer, then split and gate in torch
    plain = torch.zeros((B, 2 * inter), dtype=torch.bfloat16, device="cuda")
    mq.StackProgram([(gu, X, plain)], r, B).run()
    torch.cuda.synchronize()
    t = plain.view(B, inter // 8, 2, 8)
    gate, up = t[:, :, 0].reshape(B, inter), t[:, :, 1].reshape(B, inter)
    want = (torch.nn.functional.silu(gate.float()).to(torch.bfloat16).float() * up.float()).to(torch.bfloat16)
    assert torch.isfinite(act.float()).all()
    # same fp32 sums up to summation order -> bf16 inputs may differ by an ulp
    assert rel_err(act.float().cpu().numpy(), want.float().cpu().numpy()) <= 1e-2
    y_ref = torch.zeros_like(Y)
    mq.StackProgram([(down, act, y_ref)], r, B).run()
    torch.cuda.synchronize()
    assert torch.isfinite(Y.float()).all()
    assert rel_err(Y.float().cpu().numpy(), y_ref.float().cpu().numpy()) <= 1e-2


def test_c3_unfused_heterogeneous_plans_at_every_batch(model):
    """The 224-linear C3 config (3.5-bit budget, unfused): the per-layer-r K3S plan fits at
    B = 1, 4, 8 (the small-layer CTA-pair rule respects the staging budget, which counts the
    224-entry layer table), agrees with the per-layer graph, and the default dispatch takes
    K3S only at B <= 2 (measured, scripts/hetero_matrix.py)."""
    from paper_2602_03537_b200.config import budget_config

    cfg = budget_config(3.5, shape=model.LLAMA31_8B, seed=0, mutations=200).assignment
    stack = model.LinearStack(model.LLAMA31_8B, batch=1, fused=False)
    g = torch.Generator(device="cuda").manual_seed(31)
    for B in (1, 4, 8):
        stack.set_batch(B)
        x0 = torch.randn(B, 4096, device="cuda", generator=g).to(torch.bfloat16) * 0.5
        stack.capture(cfg, stack_kernel=True)
        assert stack.launches_per_step() == 1
        y, _ = _step(stack, x0)
        stack.capture(cfg, stack_kernel=False)
        y_ref, _ = _step(stack, x0)
        assert torch.isfinite(y.float()).all() and torch.isfinite(y_ref.float()).all()
        # two summation orders diverge by bf16 roundings compounded over 224 chained layers
        # (each layer's own parity is tested against the oracle elsewhere): 3.06e-2 seen at B = 4
        assert rel_err(y.float().cpu().numpy(), y_ref.float().cpu().numpy()) <= 6e-2, B
        assert stack.stack_kernel_ok(cfg) == (B <= 2)
