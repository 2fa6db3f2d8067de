"""Full-model decode harness: a Llama-3.1-8B-shaped decoder
whose linears are sliced ``MatLinear`` layers, so the decode number can be set
beside the paper's full-model measurement (Llama-3.1-8B-Instruct single-token
forward: 138.0 / 124.4 / 109.3 tok/s at 2 / 3 / 4 bits on an
RTX A6000).

Everything around the hot path is plain bf16 torch and is NOT part of the
deliverable: embedding lookup, RMSNorm, rotary embedding, a KV cache with
grouped-query attention (torch SDPA), SiLU gating, residuals, and a bf16
``lm_head``.  The projections (q/k/v fused, o, gate/up fused, down) are int8
parents sliced on the fly by K3 (decode) -- per layer a bit-width, uniform or
from an EvoPress-style config.  One decode step = one token for every sequence
in the batch at a fixed context length, replayed as one CUDA graph.
Weights are random (no checkpoints in this environment); the work is that of
the real model.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F

from .device import PlaneTensor
from .model import LLAMA31_8B, DecoderShape, _gain_matched_scales, full_layer_dims
from .module import MatLinear

__all__ = ["LlamaDecoder"]


def _rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * w).to(x.dtype)


def _rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    x1, x2 = x[..., : x.shape[-1] // 2], x[..., x.shape[-1] // 2:]
    return torch.cat((x1 * cos - x2 * sin, x2 * cos + x1 * sin), dim=-1)


class LlamaDecoder:
    def __init__(self, shape: DecoderShape = LLAMA31_8B, batch: int = 1, context: int = 256,
                 bits=4, vocab: int = 128256, seed: int = 0, n_layers: int | None = None):
        self.shape, self.B, self.T = shape, batch, context
        self.n_layers = n_layers or shape.n_layers
        dev = torch.device("cuda")
        g = torch.Generator(device="cuda").manual_seed(seed)
        h, hd = shape.hidden, shape.head_dim
        self.embed = (torch.randn(vocab, h, device=dev, generator=g) * 0.02).to(torch.bfloat16)
        self.lm_head = (torch.randn(vocab, h, device=dev, generator=g) / math.sqrt(h)).to(torch.bfloat16)
        self.final_norm = torch.ones(h, device=dev)
        self.blocks = []
        for i in range(self.n_layers):
            blk = {}
            for kind in ("qkv", "o", "gate_up", "down"):
                N, K = full_layer_dims(shape, kind)
                pt = PlaneTensor.random_parent(N, K, seed=seed * 7919 + i * 4 + ("qkv", "o", "gate_up", "down").index(kind),
                                               scale_range=_gain_matched_scales(K))
                blk[kind] = MatLinear(pt, 4, name="layers.%d.%s" % (i, kind))
            blk["ln1"] = torch.ones(h, device=dev)
            blk["ln2"] = torch.ones(h, device=dev)
            # KV cache filled with random history (context positions 0..T-1)
            blk["k"] = (torch.randn(batch, shape.n_kv_heads, context, hd, device=dev, generator=g)).to(torch.bfloat16)
            blk["v"] = (torch.randn(batch, shape.n_kv_heads, context, hd, device=dev, generator=g)).to(torch.bfloat16)
            self.blocks.append(blk)
        self.set_bits(bits)
        inv = 1.0 / (500000.0 ** (torch.arange(0, hd, 2, device=dev, dtype=torch.float32) / hd))
        ang = context * inv  # the decoded token sits at position `context`
        self.cos = ang.cos().to(torch.bfloat16)
        self.sin = ang.sin().to(torch.bfloat16)
        self.tokens = torch.zeros(batch, dtype=torch.long, device=dev)
        self.logits = torch.empty(batch, vocab, device=dev, dtype=torch.bfloat16)
        self.stream = torch.cuda.Stream()
        self.graph = None

    def set_bits(self, bits) -> None:
        """Uniform int, or {name: r} over the fused linears' names."""
        for i, blk in enumerate(self.blocks):
            for kind in ("qkv", "o", "gate_up", "down"):
                r = bits if isinstance(bits, int) else bits["layers.%d.%s" % (i, kind)]
                blk[kind].set_bits(r)
        self.graph = None

    def linear_bytes(self) -> int:
        from .device import algorithmic_bytes

        tot = 0
        for blk in self.blocks:
            for kind in ("qkv", "o", "gate_up", "down"):
                m = blk[kind]
                tot += algorithmic_bytes(m.planes.N, m.planes.K, self.B, m.bits, m.planes.planes_read(m.bits))
        return tot

    def _forward(self) -> None:
        s = self.shape
        B, hd = self.B, s.head_dim
        nh, nkv = s.n_heads, s.n_kv_heads
        x = self.embed[self.tokens]                                   # (B, h)
        for blk in self.blocks:
            hn = _rms_norm(x, blk["ln1"])
            qkv = blk["qkv"](hn)                                      # (B, (nh + 2 nkv) hd)
            q = qkv[:, : nh * hd].view(B, nh, 1, hd)
            k = qkv[:, nh * hd:(nh + nkv) * hd].view(B, nkv, 1, hd)
            v = qkv[:, (nh + nkv) * hd:].view(B, nkv, 1, hd)
            q = _rope(q, self.cos, self.sin)
            k = _rope(k, self.cos, self.sin)
            # attend over the cached context + the new token (the cache is not grown:
            # a fixed-length step, so the graph replays identical work)
            kk = torch.cat((blk["k"], k), dim=2)
            vv = torch.cat((blk["v"], v), dim=2)
            att = F.scaled_dot_product_attention(q, kk, vv, enable_gqa=True)   # (B, nh, 1, hd)
            x = x + blk["o"](att.reshape(B, nh * hd))
            hn = _rms_norm(x, blk["ln2"])
            gu = blk["gate_up"](hn)
            inter = s.intermediate
            x = x + blk["down"](F.silu(gu[:, :inter]) * gu[:, inter:])
        x = _rms_norm(x, self.final_norm)
        torch.matmul(x, self.lm_head.t(), out=self.logits)

    def capture(self) -> None:
        with torch.cuda.stream(self.stream):
            self._forward()  # warm up the launch paths (workspaces, cuBLAS handles)
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            self._forward()
        self.graph = g

    def step(self) -> None:
        if self.graph is None:
            self.capture()
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def decode(self, tokens_host: torch.Tensor) -> torch.Tensor:
        """One decode step through the public API: host token ids -> device ->
        the captured step -> next-token ids back on the host (greedy)."""
        if self.graph is None:
            self.capture()
        with torch.cuda.stream(self.stream):
            self.tokens.copy_(tokens_host, non_blocking=True)
            self.graph.replay()
            nxt = self.logits.argmax(-1).to("cpu", non_blocking=True)
        return nxt
