"""Full-model decode harness (BASELINE C5): a Llama /
Qwen3 / Phi-3-shaped decoder whose linears are sliced ``MatLinear`` layers, so
the decode number can be set beside the paper's full-model measurement
(Llama-3.1-8B-Instruct single-token forward: 138.0 / 124.4 /
109.3 tok/s at 2 / 3 / 4 bits on an RTX A6000), on one GPU or tensor-parallel
(``tp``: tp.decoder_plan shards of the single-GPU parents, attention over the
rank's own heads, one all-reduce after o and after down).

Everything around the hot path is NOT part of the deliverable: embedding
lookup, RMSNorm, rotary embedding, a KV cache with grouped-query attention,
SiLU gating, residuals, and a bf16 ``lm_head``.  ``glue="cuda"`` (default)
runs them as libmatq kernels: with ``linears="k3s"`` the residual add +
RMSNorm and the SiLU gating are fused into the K3S segments' activation
staging, and one ``mq_attn_decode`` launch per layer does the rotary step,
the KV-cache write and single-query GQA attention; ``glue="torch"`` is the
plain-torch statement of the same step (torch SDPA), which the tests compare
against.  The projections (q/k/v fused, o, gate/up fused, down) are int8
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
                 bits=4, vocab: int = 128256, seed: int = 0, n_layers: int | None = None, glue: str = "cuda",
                 tp: int = 1, rank: int = 0, process_group=None, linears: str | None = None):
        if glue not in ("cuda", "torch"):
            raise ValueError("glue must be 'cuda' or 'torch'")
        # "k3s": per block ONE persistent launch for o -> gate_up -> down -> next qkv with the
        # residual add + RMSNorm and the SiLU gating fused into the layers' activation staging
        # (single GPU, B <= 4); "k3": per-layer GEMV launches + the glue kernels
        if linears is None:
            linears = "k3s" if (tp == 1 and batch <= 4 and glue == "cuda") else "k3"
        if linears not in ("k3", "k3s") or (linears == "k3s" and (tp > 1 or glue != "cuda")):
            raise ValueError("linears must be 'k3' or 'k3s' (k3s: single GPU, CUDA glue)")
        self.linears = linears
        self.shape, self.B, self.T, self.glue = shape, batch, context, glue
        self.tp, self.rank, self.pg = tp, rank, process_group
        self.n_layers = n_layers or shape.n_layers
        dev = torch.device("cuda", torch.cuda.current_device())
        g = torch.Generator(device="cuda").manual_seed(seed)
        h, hd = shape.hidden, shape.head_dim
        self.embed = (torch.randn(vocab, h, device=dev, generator=g) * 0.02).to(torch.bfloat16)
        self.lm_head = (torch.randn(vocab, h, device=dev, generator=g) / math.sqrt(h)).to(torch.bfloat16)
        self.final_norm = torch.ones(h, device=dev)
        # this rank's heads: q heads [q0, q1), kv heads [k0, k1) (tp.decoder_plan)
        if tp > 1:
            from .tp import decoder_plan

            (qa, qb), (ka, kb), _ = decoder_plan(shape, "qkv", tp, rank).segments
            q0, q1, k0, k1 = qa // hd, qb // hd, (ka - shape.q_out) // hd, (kb - shape.q_out) // hd
        else:
            q0, q1, k0, k1 = 0, shape.n_heads, 0, shape.n_kv_heads
        self.nh, self.nkv = q1 - q0, k1 - k0
        grp = shape.n_heads // shape.n_kv_heads
        # local kv head of each local q head (GQA; replicated kv heads when tp does not divide them)
        self.kv_of_q = torch.tensor([(q0 + i) // grp - k0 for i in range(self.nh)], device=dev)
        self.kv_of_q32 = self.kv_of_q.to(torch.int32)
        self.uniform_gqa = self.nh % max(1, self.nkv) == 0 and all(
            (q0 + i) // grp - k0 == i // (self.nh // self.nkv) for i in range(self.nh))
        self.blocks = []
        for i in range(self.n_layers):
            blk = {}
            for kind in ("qkv", "o", "gate_up", "down"):
                N, K = full_layer_dims(shape, kind)
                sd = seed * 7919 + i * 4 + ("qkv", "o", "gate_up", "down").index(kind)
                if tp > 1:
                    from .tp import decoder_plan

                    codes, scales = PlaneTensor.random_parent_codes(N, K, 128, sd, _gain_matched_scales(K), True)
                    plan = decoder_plan(shape, kind, tp, rank)
                    rows = torch.cat([torch.arange(a, b_, device=dev) for a, b_ in plan.segments])
                    (c0, c1), (g0, g1) = plan.cols, plan.groups
                    pt = PlaneTensor.from_codes(codes[rows, c0:c1].contiguous(), 8,
                                                scales[rows, g0:g1].contiguous(), 128)
                    del codes, scales
                elif kind == "gate_up" and linears == "k3s":
                    # K3S computes silu(gate) * up where the rows finish (MQ_YOP_SILU_PAIRS): the
                    # fused parent is stored interleaved, 8 gate rows then their 8 up rows per
                    # 16-row tile (the same weights, another row order)
                    codes, scales = PlaneTensor.random_parent_codes(N, K, 128, sd, _gain_matched_scales(K), True)
                    perm = self._glu_rows(N // 2, dev)
                    pt = PlaneTensor.from_codes(codes[perm].contiguous(), 8, scales[perm].contiguous(), 128)
                    del codes, scales
                else:
                    pt = PlaneTensor.random_parent(N, K, seed=sd, scale_range=_gain_matched_scales(K),
                                                   signed_rows=True)
                blk[kind] = MatLinear(pt, 4, name="layers.%d.%s" % (i, kind))
            blk["ln1"] = torch.ones(h, device=dev)
            blk["ln2"] = torch.ones(h, device=dev)
            if shape.qk_norm:
                blk["qn"] = 1.0 + 0.1 * torch.randn(hd, device=dev, generator=g)
                blk["kn"] = 1.0 + 0.1 * torch.randn(hd, device=dev, generator=g)
            # KV cache (the rank's kv heads): random history at positions 0..T-1, the decoded
            # token's k/v at T
            blk["kc"] = torch.zeros(batch, self.nkv, context + 1, hd, device=dev, dtype=torch.bfloat16)
            blk["vc"] = torch.zeros_like(blk["kc"])
            hk = torch.randn(batch, shape.n_kv_heads, context, hd, device=dev, generator=g)
            hv = torch.randn(batch, shape.n_kv_heads, context, hd, device=dev, generator=g)
            blk["kc"][:, :, :context] = hk[:, k0:k1]
            blk["vc"][:, :, :context] = hv[:, k0:k1]
            blk["k"], blk["v"] = blk["kc"][:, :, :context], blk["vc"][:, :, :context]
            self.blocks.append(blk)
        self.set_bits(bits)
        inv = 1.0 / (500000.0 ** (torch.arange(0, hd, 2, device=dev, dtype=torch.float32) / hd))
        ang = context * inv  # the decoded token sits at position `context`
        self.cos = ang.cos().to(torch.bfloat16)
        self.sin = ang.sin().to(torch.bfloat16)
        self.tokens = torch.zeros(batch, dtype=torch.long, device=dev)
        self.logits = torch.empty(batch, vocab, device=dev, dtype=torch.bfloat16)
        nq = self.nh * hd
        inter = self.blocks[0]["down"].planes.K
        self.inter = inter
        e = lambda *sz: torch.empty(*sz, device=dev, dtype=torch.bfloat16)  # noqa: E731
        self.buf = {"x": e(batch, h), "hn": e(batch, h), "qkv": e(batch, nq + 2 * self.nkv * hd),
                    "q": e(batch, self.nh, 1, hd), "o": e(batch, h), "gu": e(batch, 2 * inter),
                    "act": e(batch, inter), "d": e(batch, h), "att": e(batch, nq), "xr": e(batch, h)}
        self.stream = torch.cuda.Stream()
        self.graph = None
        self.segments = None

    @staticmethod
    def _glu_rows(inter: int, dev) -> torch.Tensor:
        """Row order of an interleaved gate/up parent: per 16-row tile, gate rows 8t..8t+7
        then up rows inter + 8t .. inter + 8t + 7."""
        t = torch.arange(inter // 8, device=dev).repeat_interleave(8) * 8 + torch.arange(8, device=dev).repeat(inter // 8)
        return torch.stack((t.view(-1, 8), (t + inter).view(-1, 8)), dim=1).reshape(-1)

    @property
    def gate_up_rows(self):
        """The gate_up parent's row order (None: [gate | up]), for references that decode it."""
        if self.linears != "k3s":
            return None
        return self._glu_rows(self.inter, self.embed.device)

    def _all_reduce(self, t: torch.Tensor) -> None:
        if self.tp > 1:
            torch.distributed.all_reduce(t, group=self.pg)

    def _qk_norm(self, blk) -> None:
        """Qwen3: per-head RMSNorm of q and k (in the fused qkv row) before the rotary step."""
        if not self.shape.qk_norm:
            return
        B, hd = self.B, self.shape.head_dim
        qk = self.buf["qkv"][:, : (self.nh + self.nkv) * hd].view(B, self.nh + self.nkv, hd)
        w = torch.cat((blk["qn"].expand(self.nh, hd), blk["kn"].expand(self.nkv, hd)))
        qk.copy_(_rms_norm(qk, w, 1e-6))

    def _attend(self, q, kc, vc):
        """Single-query attention over the cache with the rank's GQA head map."""
        if self.uniform_gqa:
            return F.scaled_dot_product_attention(q, kc, vc, enable_gqa=True)
        return F.scaled_dot_product_attention(q, kc.index_select(1, self.kv_of_q),
                                              vc.index_select(1, self.kv_of_q))

    def _attn_decode(self, blk, st) -> None:
        """(q/k RMSNorm +) rotary step, KV-cache write at position T and single-query
        attention for every q head in one kernel (mq_attn_decode) -> buf['att']."""
        from . import _lib

        s, b = self.shape, self.buf
        qn = _lib.ptr(blk["qn"]) if s.qk_norm else None
        kn = _lib.ptr(blk["kn"]) if s.qk_norm else None
        _lib.call("mq_attn_decode", _lib.ptr(b["qkv"]), _lib.ptr(self.cos), _lib.ptr(self.sin), qn, kn, 1e-6,
                  _lib.ptr(blk["kc"]), _lib.ptr(blk["vc"]), _lib.ptr(self.kv_of_q32), _lib.ptr(b["att"]),
                  self.B, self.nh, self.nkv, s.head_dim, self.T + 1, self.T, st)

    def set_bits(self, bits) -> None:
        """Uniform int, or {name: r} over the fused linears' names."""
        for i, blk in enumerate(self.blocks):
            for kind in ("qkv", "o", "gate_up", "down"):
                r = bits if isinstance(bits, int) else bits["layers.%d.%s" % (i, kind)]
                blk[kind].set_bits(r)
        self.graph = None
        self.segments = None

    def _build_segments(self) -> None:
        """K3S programs: block i's [o_i, gate_up_i (+ x += o; RMSNorm ln2; SiLU gating of
        its interleaved rows as it writes them), down_i, qkv_{i+1} (+ x += down; RMSNorm ln1
        of block i+1; x written back)]; the last block writes its post-attention residual
        to buf['xr'] for the final norm."""
        from . import _lib
        from .device import StackProgram

        b, h, nb = self.buf, self.shape.hidden, len(self.blocks)
        self.segments = []
        for i, blk in enumerate(self.blocks):
            layers = [(blk["o"].planes, b["att"], b["o"]), (blk["gate_up"].planes, b["o"], b["act"]),
                      (blk["down"].planes, b["act"], b["d"])]
            rs = [blk["o"].bits, blk["gate_up"].bits, blk["down"].bits]
            last = i == nb - 1
            ops = [None,
                   dict(xop=_lib.MQ_XOP_ADD_RMSNORM, res_in=b["x"], res_out=b["xr"] if last else None,
                        norm_w=blk["ln2"], eps=1e-5, yop=_lib.MQ_YOP_SILU_PAIRS),
                   None]
            if not last:
                nxt = self.blocks[i + 1]
                layers.append((nxt["qkv"].planes, b["d"], b["qkv"]))
                rs.append(nxt["qkv"].bits)
                ops.append(dict(xop=_lib.MQ_XOP_ADD_RMSNORM, res_in=None, res_out=b["x"],
                                norm_w=nxt["ln1"], eps=1e-5))
            self.segments.append(StackProgram(layers, rs[0] if len(set(rs)) == 1 else rs, self.B, ops=ops))

    def linear_bytes(self) -> int:
        from .device import algorithmic_bytes

        tot = 0
        for blk in self.blocks:
            for kind in ("qkv", "o", "gate_up", "down"):
                m = blk[kind]
                tot += algorithmic_bytes(m.planes.N, m.planes.K, self.B, m.bits, m.planes.planes_read(m.bits))
        return tot

    def _forward(self) -> None:
        if self.glue != "cuda":
            self._forward_torch()
        elif self.linears == "k3s":
            self._forward_k3s()
        else:
            self._forward_fused()

    def _forward_k3s(self, parts=("linear", "attn", "glue", "comm", "head")) -> None:
        """One decode step with one K3S launch per block (o, gate_up, down and the
        next block's qkv; the residual / RMSNorm / SiLU glue fused into staging):
        per block K3S + one attention kernel (rotary, KV write, single-query attention)."""
        from . import _lib

        if self.segments is None:
            self._build_segments()
        s = self.shape
        B, hd, T = self.B, s.head_dim, self.T
        nh, nkv, h = self.nh, self.nkv, s.hidden
        b = self.buf
        st = _lib.stream_ptr(None)
        lin, attn, glue, head = ("linear" in parts), ("attn" in parts), ("glue" in parts), ("head" in parts)
        if head:
            torch.index_select(self.embed, 0, self.tokens, out=b["x"])
        blk0 = self.blocks[0]
        if glue:
            _lib.call("mq_add_rmsnorm", _lib.ptr(b["x"]), None, _lib.ptr(blk0["ln1"]), _lib.ptr(b["hn"]),
                      B, h, 1e-5, st)
        if lin:
            blk0["qkv"].planes.linear(b["hn"], blk0["qkv"].bits, out=b["qkv"], pdl=True)
        for i, blk in enumerate(self.blocks):
            if attn:
                self._attn_decode(blk, st)
            if lin:
                self.segments[i].run(torch.cuda.current_stream())
        if glue:
            _lib.call("mq_add_rmsnorm", _lib.ptr(b["xr"]), _lib.ptr(b["d"]), _lib.ptr(self.final_norm),
                      _lib.ptr(b["hn"]), B, h, 1e-5, st)
        if head:
            torch.matmul(b["hn"], self.lm_head.t(), out=self.logits)

    PARTS = ("linear", "attn", "glue", "comm", "head")

    def _forward_fused(self, parts=PARTS) -> None:
        """One decode step: 4 sliced linears (PDL-chained K3) + 2 glue kernels
        (norm, gating) + one attention kernel (rotary, KV write, attention) per block (+ 2 all-reduces
        under tensor parallelism).  ``parts`` keeps only some component
        classes (component_ms times each alone on the same buffers)."""
        from . import _lib

        s = self.shape
        B, hd, T = self.B, s.head_dim, self.T
        nh, nkv, h = self.nh, self.nkv, s.hidden
        b = self.buf
        st = _lib.stream_ptr(None)
        lin, attn, glue, comm, head = (p in parts for p in self.PARTS)
        if head:
            torch.index_select(self.embed, 0, self.tokens, out=b["x"])
        delta = None
        for blk in self.blocks:
            if glue:
                _lib.call("mq_add_rmsnorm", _lib.ptr(b["x"]), _lib.ptr(delta) if delta is not None else None,
                          _lib.ptr(blk["ln1"]), _lib.ptr(b["hn"]), B, h, 1e-5, st)
            if lin:
                blk["qkv"].planes.linear(b["hn"], blk["qkv"].bits, out=b["qkv"], pdl=True)
            if attn:
                self._attn_decode(blk, st)
            if lin:
                blk["o"].planes.linear(b["att"], blk["o"].bits, out=b["o"], pdl=True)
            if comm:
                self._all_reduce(b["o"])
            if glue:
                _lib.call("mq_add_rmsnorm", _lib.ptr(b["x"]), _lib.ptr(b["o"]), _lib.ptr(blk["ln2"]),
                          _lib.ptr(b["hn"]), B, h, 1e-5, st)
            if lin:
                blk["gate_up"].planes.linear(b["hn"], blk["gate_up"].bits, out=b["gu"], pdl=True)
            if glue:
                _lib.call("mq_silu_mul", _lib.ptr(b["gu"]), _lib.ptr(b["act"]), B, self.inter, st)
            if lin:
                blk["down"].planes.linear(b["act"], blk["down"].bits, out=b["d"], pdl=True)
            if comm:
                self._all_reduce(b["d"])
            delta = b["d"]
        if glue:
            _lib.call("mq_add_rmsnorm", _lib.ptr(b["x"]), _lib.ptr(delta), _lib.ptr(self.final_norm),
                      _lib.ptr(b["hn"]), B, h, 1e-5, st)
        if head:
            torch.matmul(b["hn"], self.lm_head.t(), out=self.logits)

    def component_ms(self, reps: int = 20) -> dict:
        """Per-component device time of one step (ms): each component class
        captured alone in its own CUDA graph (same shapes and buffers), plus
        the whole step.  Under TP, "comm" is the all-reduces."""
        def time_graph(fn):
            self.stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.stream):
                fn()
            self.stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                fn()
            with torch.cuda.stream(self.stream):
                g.replay()
            self.stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            with torch.cuda.stream(self.stream):
                for _ in range(reps):
                    g.replay()
            e1.record(self.stream)
            e1.synchronize()
            return e0.elapsed_time(e1) / reps

        fwd = self._forward_k3s if self.linears == "k3s" else self._forward_fused
        out = {"step": time_graph(lambda: fwd()), "linears": self.linears}
        for part in self.PARTS:
            if part == "comm" and self.tp == 1:
                continue
            out[part] = time_graph(lambda p=part: fwd(parts=(p,)))
        out["sum_of_parts"] = sum(v for k, v in out.items() if k not in ("step", "linears"))
        return out

    def _forward_torch(self) -> None:
        s = self.shape
        B, hd = self.B, s.head_dim
        nh, nkv = self.nh, self.nkv
        x = self.embed[self.tokens]                                   # (B, h)
        for blk in self.blocks:
            hn = _rms_norm(x, blk["ln1"])
            qkv = blk["qkv"](hn)                                      # (B, (nh + 2 nkv) hd)
            if s.qk_norm:
                qk = qkv[:, : (nh + nkv) * hd].view(B, nh + nkv, hd)
                w = torch.cat((blk["qn"].expand(nh, hd), blk["kn"].expand(nkv, hd)))
                qkv = torch.cat((_rms_norm(qk, w, 1e-6).reshape(B, -1), qkv[:, (nh + nkv) * hd:]), dim=1)
            q = qkv[:, : nh * hd].view(B, nh, 1, hd)
            k = qkv[:, nh * hd:(nh + nkv) * hd].view(B, nkv, 1, hd)
            v = qkv[:, (nh + nkv) * hd:].view(B, nkv, 1, hd)
            q = _rope(q, self.cos, self.sin)
            k = _rope(k, self.cos, self.sin)
            # attend over the cached context + the new token (the cache is not grown:
            # a fixed-length step, so the graph replays identical work)
            kk = torch.cat((blk["k"], k), dim=2)
            vv = torch.cat((blk["v"], v), dim=2)
            att = self._attend(q, kk, vv)                             # (B, nh, 1, hd)
            o = blk["o"](att.reshape(B, nh * hd))
            self._all_reduce(o)
            x = x + o
            hn = _rms_norm(x, blk["ln2"])
            gu = blk["gate_up"](hn)
            inter = self.inter
            d = blk["down"](F.silu(gu[:, :inter]) * gu[:, inter:])
            self._all_reduce(d)
            x = x + d
        x = _rms_norm(x, self.final_norm)
        torch.matmul(x, self.lm_head.t(), out=self.logits)

    def capture(self, graph: bool = True) -> None:
        # the buffers (tokens, KV cache, ...) were initialised on the caller's stream: without
        # this wait a fresh decoder could embed stale token ids (seen with a second decoder in
        # one process: an index_select device assert)
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            self._forward()  # warm up the launch paths (workspaces, cuBLAS handles)
        self.stream.synchronize()
        if not graph:  # e.g. gloo collectives, which cannot be graph-captured
            self.graph = False
            return
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            self._forward()
        self.graph = g

    def step(self) -> None:
        if self.graph is None:
            self.capture()
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            if self.graph is False:
                self._forward()
            else:
                self.graph.replay()

    def decode(self, tokens_host: torch.Tensor) -> torch.Tensor:
        """One decode step through the public API: host token ids -> device ->
        the captured step -> next-token ids back on the host (greedy)."""
        if self.graph is None:
            self.capture()
        with torch.cuda.stream(self.stream):
            self.tokens.copy_(tokens_host, non_blocking=True)
            if self.graph is False:
                self._forward()
            else:
                self.graph.replay()
            nxt = self.logits.argmax(-1).to("cpu", non_blocking=True)
        return nxt
