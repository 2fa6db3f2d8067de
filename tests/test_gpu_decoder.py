"""Full-model decode harness (BASELINE C5) beyond glue-vs-glue:

* the fused CUDA step against an fp32 statement of the decoder computed from
  the DEQUANTISED weights (PlaneTensor.decode: the reference's dequantise-then-
  matmul, matmul.py:85-92), every intermediate in fp32;
* Qwen3-style per-head q / k RMSNorm (shapes.QWEN3_14B.qk_norm) and Phi-3-style
  GQA through both glue paths;
* tensor parallelism: two ranks sharing the one GPU over gloo against the
  single-GPU decoder with the same seed (tp.decoder_plan shards, replicated kv
  heads at tp = 2 for a 1-kv-head config).
"""

import math
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
import torch.nn.functional as F

from tests.conftest import rel_err

pytestmark = pytest.mark.gpu

TINY = dict(name="tiny", hidden=512, intermediate=1024, n_heads=8, n_kv_heads=2, head_dim=64, n_layers=2)


@pytest.fixture(scope="module")
def llama():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_03537_b200 import llama as m

    return m


def _shape(**kw):
    from paper_2602_03537_b200.shapes import DecoderShape

    d = dict(TINY)
    d.update(kw)
    return DecoderShape(**d)


def _fp32_reference(dec, r):
    """fp32 decoder step from dequantised weights (no bf16 rounding anywhere)."""
    s = dec.shape
    B, hd, nh, nkv = dec.B, s.head_dim, dec.nh, dec.nkv

    def rms(x, w, eps=1e-5):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w

    def rope(x):
        c, sn = dec.cos.float(), dec.sin.float()
        x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
        return torch.cat((x1 * c - x2 * sn, x2 * c + x1 * sn), dim=-1)

    x = dec.embed[dec.tokens].float()
    for blk in dec.blocks:
        W = {k: blk[k].planes.decode(r) for k in ("qkv", "o", "gate_up", "down")}
        perm = dec.gate_up_rows  # k3s decoders store gate/up interleaved (MQ_YOP_SILU_PAIRS)
        if perm is not None:
            std = torch.empty_like(W["gate_up"])
            std[perm] = W["gate_up"]
            W["gate_up"] = std
        qkv = rms(x, blk["ln1"]) @ W["qkv"].t()
        if s.qk_norm:
            qk = qkv[:, : (nh + nkv) * hd].view(B, nh + nkv, hd)
            w = torch.cat((blk["qn"].expand(nh, hd), blk["kn"].expand(nkv, hd)))
            qkv = torch.cat((rms(qk, w, 1e-6).reshape(B, -1), qkv[:, (nh + nkv) * hd:]), dim=1)
        q = rope(qkv[:, : nh * hd].view(B, nh, 1, hd))
        k = rope(qkv[:, nh * hd:(nh + nkv) * hd].view(B, nkv, 1, hd))
        v = qkv[:, (nh + nkv) * hd:].view(B, nkv, 1, hd)
        kk = torch.cat((blk["k"].float(), k), dim=2).index_select(1, dec.kv_of_q)
        vv = torch.cat((blk["v"].float(), v), dim=2).index_select(1, dec.kv_of_q)
        att = torch.softmax((q @ kk.transpose(-1, -2)) / math.sqrt(hd), dim=-1) @ vv
        x = x + att.reshape(B, nh * hd) @ W["o"].t()
        gu = rms(x, blk["ln2"]) @ W["gate_up"].t()
        inter = dec.inter
        x = x + (F.silu(gu[:, :inter]) * gu[:, inter:]) @ W["down"].t()
    return rms(x, dec.final_norm) @ dec.lm_head.float().t()


@pytest.mark.parametrize("linears", ["k3", "k3s"])
@pytest.mark.parametrize("qk_norm", [False, True], ids=["llama-gqa", "qwen3-qknorm"])
@pytest.mark.parametrize("r", [4, 8])
def test_decoder_step_vs_fp32_dequantised_reference(llama, qk_norm, r, linears):
    """linears = k3s: one persistent launch per block with the residual add +
    RMSNorm and the SiLU gating fused into the layers' activation staging."""
    shape = _shape(qk_norm=qk_norm)
    dec = llama.LlamaDecoder(shape, batch=3, context=16, bits=r, vocab=1024, linears=linears)
    dec.tokens.copy_(torch.tensor([1, 77, 500], device="cuda"))
    with torch.cuda.stream(dec.stream):
        dec._forward()
    dec.stream.synchronize()
    want = _fp32_reference(dec, r)
    got = dec.logits.float()
    assert torch.isfinite(got).all()
    assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 3e-2


def test_qk_norm_fused_matches_torch_glue(llama):
    outs = {}
    for glue in ("cuda", "torch"):
        dec = llama.LlamaDecoder(_shape(qk_norm=True), batch=2, context=16, bits=4, vocab=1024, glue=glue)
        dec.tokens.copy_(torch.tensor([3, 9], device="cuda"))
        with torch.cuda.stream(dec.stream):
            dec._forward()
        dec.stream.synchronize()
        outs[glue] = dec.logits.float().clone()
    assert rel_err(outs["cuda"].cpu().numpy(), outs["torch"].cpu().numpy()) <= 2e-2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tp_worker(rank, world, port, kv, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_03537_b200.llama import LlamaDecoder
        from tests.conftest import rel_err as re

        shape = _shape(n_kv_heads=kv)
        dec = LlamaDecoder(shape, batch=2, context=16, bits=4, vocab=1024, tp=world, rank=rank,
                           process_group=dist.group.WORLD)
        dec.capture(graph=False)
        dec.tokens.copy_(torch.tensor([4, 40], device="cuda"))
        torch.cuda.synchronize()
        dec.step()
        torch.cuda.synchronize()
        if rank == 0:
            ref = LlamaDecoder(shape, batch=2, context=16, bits=4, vocab=1024)
            ref.tokens.copy_(torch.tensor([4, 40], device="cuda"))
            torch.cuda.synchronize()
            ref.step()
            torch.cuda.synchronize()
            q.put((kv, dec.nh, dec.nkv, re(dec.logits.float().cpu().numpy(), ref.logits.float().cpu().numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kv", [2, 1], ids=["kv-split", "kv-replicated"])
def test_decoder_tp2_gloo_matches_single_gpu(llama, kv):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, kv, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    kv_, nh, nkv, err = q.get()
    assert nh == 4 and nkv == (1 if kv == 2 else 1)
    assert err <= 3e-2, err


@pytest.mark.parametrize("B", [1, 4])
def test_decoder_k3s_segments_match_per_layer_path(llama, B):
    """The fused K3S block segments against the per-layer K3 + glue-kernel step
    (same weights): only summation orders differ; graph replays are bitwise stable."""
    outs = {}
    for lin in ("k3", "k3s"):
        dec = llama.LlamaDecoder(_shape(), batch=B, context=16, bits=4, vocab=1024, linears=lin)
        dec.tokens.copy_(torch.arange(B, device="cuda") * 13 + 1)
        torch.cuda.synchronize()
        dec.step()
        torch.cuda.synchronize()
        outs[lin] = dec.logits.float().clone()
        if lin == "k3s":
            assert len(dec.segments) == dec.n_layers
            dec.step()
            torch.cuda.synchronize()
            assert torch.equal(dec.logits.float(), outs[lin])
    assert rel_err(outs["k3s"].cpu().numpy(), outs["k3"].cpu().numpy()) <= 2e-2


@pytest.mark.parametrize("hd", [64, 128])
@pytest.mark.parametrize("qk_norm", [False, True], ids=["plain", "qknorm"])
@pytest.mark.parametrize("heads", [(8, 2, None), (6, 3, [0, 0, 1, 1, 1, 2])], ids=["gqa", "ragged-map"])
@pytest.mark.parametrize("B,T", [(1, 1), (3, 17), (2, 300), (1, 20001)])
def test_attn_decode_kernel_vs_torch(llama, hd, qk_norm, heads, B, T):
    """mq_attn_decode (rotary + optional q/k RMSNorm + KV write + single-query
    attention, one launch) against the torch glue (_rms_norm, _rope in bf16) and an
    fp32 softmax-attention; T = 20001 takes the > 48 KB dynamic shared-memory path."""
    from paper_2602_03537_b200 import _lib

    nh, nkv, kmap = heads
    kmap = kmap or [i // (nh // nkv) for i in range(nh)]
    pos = T - 1
    g = torch.Generator(device="cuda").manual_seed(hd + T + nh)
    qkv = torch.randn(B, (nh + 2 * nkv) * hd, device="cuda", generator=g).to(torch.bfloat16)
    kc = torch.randn(B, nkv, T, hd, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(B, nkv, T, hd, device="cuda", generator=g).to(torch.bfloat16)
    kc0, vc0 = kc.clone(), vc.clone()
    ang = 37.0 / (10000.0 ** (torch.arange(0, hd, 2, device="cuda", dtype=torch.float32) / hd))
    cos, sin = ang.cos().to(torch.bfloat16), ang.sin().to(torch.bfloat16)
    qn = (1.0 + 0.1 * torch.randn(hd, device="cuda", generator=g)) if qk_norm else None
    kn = (1.0 + 0.1 * torch.randn(hd, device="cuda", generator=g)) if qk_norm else None
    kv_of_q = torch.tensor(kmap, device="cuda", dtype=torch.int32)
    att = torch.full((B, nh * hd), float("nan"), device="cuda", dtype=torch.bfloat16)
    _lib.call("mq_attn_decode", _lib.ptr(qkv), _lib.ptr(cos), _lib.ptr(sin),
              _lib.ptr(qn) if qk_norm else None, _lib.ptr(kn) if qk_norm else None, 1e-6,
              _lib.ptr(kc), _lib.ptr(vc), _lib.ptr(kv_of_q), _lib.ptr(att), B, nh, nkv, hd, T, pos,
              _lib.stream_ptr(None))
    torch.cuda.synchronize()
    q = qkv[:, : nh * hd].view(B, nh, hd)
    k = qkv[:, nh * hd:(nh + nkv) * hd].view(B, nkv, hd)
    v = qkv[:, (nh + nkv) * hd:].view(B, nkv, hd)
    if qk_norm:
        q, k = llama._rms_norm(q, qn, 1e-6), llama._rms_norm(k, kn, 1e-6)
    q, k = llama._rope(q, cos, sin), llama._rope(k, cos, sin)
    # the new k / v land at pos (rounding of the fused norm may differ by one bf16 ulp)
    assert torch.equal(vc[:, :, pos], v)
    torch.testing.assert_close(kc[:, :, pos].float(), k.float(), rtol=1e-2, atol=1e-2)
    assert torch.equal(kc[:, :, :pos], kc0[:, :, :pos]) and torch.equal(vc[:, :, :pos], vc0[:, :, :pos])
    idx = kv_of_q.long()
    kk = torch.cat((kc0[:, :, :pos].float(), k.float().unsqueeze(2)), dim=2).index_select(1, idx)
    vv = torch.cat((vc0[:, :, :pos].float(), v.float().unsqueeze(2)), dim=2).index_select(1, idx)
    p = torch.softmax((q.float().unsqueeze(2) @ kk.transpose(-1, -2)) / math.sqrt(hd), dim=-1)
    want = (p @ vv).reshape(B, nh * hd)
    got = att.float()
    assert torch.isfinite(got).all()
    assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 1e-2


def test_attn_decode_rejects_bad_shapes(llama):
    from paper_2602_03537_b200 import _lib

    x = torch.zeros(64, device="cuda", dtype=torch.bfloat16)
    m = torch.zeros(2, device="cuda", dtype=torch.int32)
    for hd, T, pos in ((96, 4, 3), (64, 4, 4), (64, 4, -1)):
        with pytest.raises(Exception):
            _lib.call("mq_attn_decode", _lib.ptr(x), _lib.ptr(x), _lib.ptr(x), None, None, 1e-6, _lib.ptr(x),
                      _lib.ptr(x), _lib.ptr(m), _lib.ptr(x), 1, 2, 1, hd, T, pos, _lib.stream_ptr(None))


def test_fresh_decoders_in_one_process(llama):
    """Decoders built one after another in one process (the caching allocator hands the
    second one the first one's memory): its buffers are initialised on the caller's
    stream, so capture / step must wait for that stream (before the fix the second
    decoder embedded stale token ids: an index_select device assert)."""
    for B in (1, 2, 3, 2):
        dec = llama.LlamaDecoder(batch=B, n_layers=2)
        for _ in range(3):
            dec.step()
        torch.cuda.synchronize()
        assert torch.isfinite(dec.logits.float()).all(), B
        del dec
        torch.cuda.empty_cache()
