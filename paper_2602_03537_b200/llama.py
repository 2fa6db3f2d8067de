"""Full-model decode harness: a Llama-3.1-8B-shaped decoder
whose linears are sliced ``MatLinear`` layers, so the decode number can be set
beside the paper's full-model measurement (Llama-3.1-8B-Instruct single-token
forward: 138.0 / 124.4 / 109.3 tok/s at 2 / 3 / 4 bits on an
RTX A6000).

Everything around the hot path is NOT part of the deliverable: embedding
lookup, RMSNorm, rotary embedding, a KV cache with grouped-query attention
(torch SDPA), SiLU gating, residuals, and a bf16 ``lm_head``.  ``glue="cuda"``
(default) runs the row-wise steps as three fused kernels from libmatq
(residual add + RMSNorm, rotary + KV-cache write, SiLU gating: 3 launches per
block instead of ~25 torch kernels; attention stays torch SDPA, which beat a
simple single-query kernel here); ``glue="torch"`` is the plain-torch
statement of the same step, which the tests compare against.  The projections (q/k/v fused, o, gate/up fused, down) are int8
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
                 bits=4, vocab: int = 128256, seed: int = 0, n_layers: int | None = None, glue: str = "cuda"):
        if glue not in ("cuda", "torch"):
            raise ValueError("glue must be 'cuda' or 'torch'")
        self.shape, self.B, self.T, self.glue = shape, batch, context, glue
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
                                               scale_range=_gain_matched_scales(K), signed_rows=True)
                blk[kind] = MatLinear(pt, 4, name="layers.%d.%s" % (i, kind))
            blk["ln1"] = torch.ones(h, device=dev)
            blk["ln2"] = torch.ones(h, device=dev)
            # KV cache: random history at positions 0..T-1, the decoded token's k/v at T
            blk["kc"] = torch.zeros(batch, shape.n_kv_heads, context + 1, hd, device=dev, dtype=torch.bfloat16)
            blk["vc"] = torch.zeros_like(blk["kc"])
            blk["kc"][:, :, :context] = torch.randn(batch, shape.n_kv_heads, context, hd, device=dev, generator=g)
            blk["vc"][:, :, :context] = torch.randn(batch, shape.n_kv_heads, context, hd, device=dev, generator=g)
            blk["k"], blk["v"] = blk["kc"][:, :, :context], blk["vc"][:, :, :context]
            self.blocks.append(blk)
        self.set_bits(bits)
        inv = 1.0 / (500000.0 ** (torch.arange(0, hd, 2, device=dev, dtype=torch.float32) / hd))
        ang = context * inv  # the decoded token sits at position `context`
        self.cos = ang.cos().to(torch.bfloat16)
        self.sin = ang.sin().to(torch.bfloat16)
        self.tokens = torch.zeros(batch, dtype=torch.long, device=dev)
        self.logits = torch.empty(batch, vocab, device=dev, dtype=torch.bfloat16)
        nq = shape.n_heads * hd
        e = lambda *sz: torch.empty(*sz, device=dev, dtype=torch.bfloat16)  # noqa: E731
        self.buf = {"x": e(batch, h), "hn": e(batch, h), "qkv": e(batch, nq + 2 * shape.n_kv_heads * hd),
                    "q": e(batch, shape.n_heads, 1, hd), "o": e(batch, h), "gu": e(batch, 2 * shape.intermediate),
                    "act": e(batch, shape.intermediate), "d": e(batch, h)}
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
        if self.glue == "cuda":
            self._forward_fused()
        else:
            self._forward_torch()

    def _forward_fused(self) -> None:
        """One decode step: 4 sliced linears (PDL-chained K3) + 3 fused glue
        kernels (norm, rotary/KV, gating) + SDPA per block."""
        from . import _lib

        s = self.shape
        B, hd, T = self.B, s.head_dim, self.T
        nh, nkv, h = s.n_heads, s.n_kv_heads, s.hidden
        b = self.buf
        st = _lib.stream_ptr(None)
        torch.index_select(self.embed, 0, self.tokens, out=b["x"])
        delta = None
        for blk in self.blocks:
            _lib.call("mq_add_rmsnorm", _lib.ptr(b["x"]), _lib.ptr(delta) if delta is not None else None,
                      _lib.ptr(blk["ln1"]), _lib.ptr(b["hn"]), B, h, 1e-5, st)
            blk["qkv"].planes.linear(b["hn"], blk["qkv"].bits, out=b["qkv"], pdl=True)
            _lib.call("mq_rope_kv", _lib.ptr(b["qkv"]), _lib.ptr(self.cos), _lib.ptr(self.sin), _lib.ptr(b["q"]),
                      _lib.ptr(blk["kc"]), _lib.ptr(blk["vc"]), B, nh, nkv, hd, T + 1, T, st)
            att = F.scaled_dot_product_attention(b["q"], blk["kc"], blk["vc"], enable_gqa=True)
            blk["o"].planes.linear(att.reshape(B, nh * hd), blk["o"].bits, out=b["o"], pdl=True)
            _lib.call("mq_add_rmsnorm", _lib.ptr(b["x"]), _lib.ptr(b["o"]), _lib.ptr(blk["ln2"]),
                      _lib.ptr(b["hn"]), B, h, 1e-5, st)
            blk["gate_up"].planes.linear(b["hn"], blk["gate_up"].bits, out=b["gu"], pdl=True)
            _lib.call("mq_silu_mul", _lib.ptr(b["gu"]), _lib.ptr(b["act"]), B, s.intermediate, st)
            blk["down"].planes.linear(b["act"], blk["down"].bits, out=b["d"], pdl=True)
            delta = b["d"]
        _lib.call("mq_add_rmsnorm", _lib.ptr(b["x"]), _lib.ptr(delta), _lib.ptr(self.final_norm),
                  _lib.ptr(b["hn"]), B, h, 1e-5, st)
        torch.matmul(b["hn"], self.lm_head.t(), out=self.logits)

    def _forward_torch(self) -> None:
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
