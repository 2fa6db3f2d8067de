"""Decode-step proxies built from sliced linears (BASELINE configs 2, 3, 5).

``LinearStack`` holds the linear layers of a Llama/Qwen/Phi-shaped decoder as
int8 parents resident in HBM (P8 planes) and runs one decode step -- every
linear of every block, in dependency order -- as a CUDA graph of K3
launches chained with programmatic dependent launch:

    x -> qkv -> (q part) -> o [-> all-reduce] -> gate_up -> (gate part) -> down [-> all-reduce] -> x

Attention, KV cache, norms, activations and lm_head are not part of the hot
path and are omitted (the numbers are labelled "linear stack").  Each layer
carries its own bit-width r (uniform or an EvoPress-style heterogeneous
config) and switching r re-captures the graph without touching the weights.

Tensor parallelism: qkv / gate_up are column-parallel (rows
split), o / down row-parallel (K split in multiples of 256) followed by one
NCCL all-reduce of the (B, hidden) partial.  ``tp = 1`` has no collective.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .device import LADDER, PlaneTensor, algorithmic_bytes, reserve_workspace


@dataclass(frozen=True)
class DecoderShape:
    name: str
    hidden: int
    intermediate: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    n_layers: int

    @property
    def qkv_out(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def q_out(self) -> int:
        return self.n_heads * self.head_dim


LLAMA31_8B = DecoderShape("Llama-3.1-8B", 4096, 14336, 32, 8, 128, 32)
QWEN3_14B = DecoderShape("Qwen3-14B", 5120, 17408, 40, 8, 128, 40)
PHI3_MEDIUM = DecoderShape("Phi-3-Medium", 5120, 17920, 40, 10, 128, 40)
SHAPES = {s.name: s for s in (LLAMA31_8B, QWEN3_14B, PHI3_MEDIUM)}

KINDS = ("qkv", "o", "gate_up", "down")


def layer_names(shape: DecoderShape) -> list[str]:
    return ["layers.%d.%s" % (i, k) for i in range(shape.n_layers) for k in KINDS]


def tp_layer_dims(shape: DecoderShape, kind: str, tp: int) -> tuple[int, int]:
    """(N, K) of one rank's shard of a fused linear."""
    h, inter = shape.hidden, shape.intermediate
    if kind == "qkv":
        return shape.qkv_out // tp, h
    if kind == "o":
        return h, shape.q_out // tp
    if kind == "gate_up":
        return 2 * inter // tp, h
    if kind == "down":
        return h, inter // tp
    raise KeyError(kind)


def _gain_matched_scales(K: int):
    """Scale range keeping activations O(1) through a random-init chain.

    |w| ~ scale * 74 (RMS of a uniform int8 parent's centred codes); a K-long
    dot product grows by sqrt(K) * 74 * scale, so centre the scale on
    1 / (74 sqrt(K)) with the reference's 4x spread (matmul.py:131 uses
    U(0.005, 0.02)).  Only the values change, not the work.
    """
    c = 1.0 / (74.0 * K ** 0.5)
    return (0.4 * c, 1.6 * c)


class LinearStack:
    def __init__(self, shape: DecoderShape = LLAMA31_8B, batch: int = 1, group_size: int = 128,
                 tp: int = 1, rank: int = 0, process_group=None, seed: int = 0,
                 n_layers: int | None = None):
        _lib.require_cuda()
        if batch < 1 or batch > 32:
            raise ValueError("decode batch must lie in [1, 32]")
        self.shape = shape
        self.B = batch
        self.G = group_size
        self.tp, self.rank, self.pg = tp, rank, process_group
        self.n_layers = n_layers or shape.n_layers
        self.layers: list[tuple[str, str, PlaneTensor]] = []
        for i in range(self.n_layers):
            for kind in KINDS:
                N, K = tp_layer_dims(shape, kind, tp)
                pt = PlaneTensor.random_parent(N, K, group_size,
                                               seed=seed * 1000003 + (i * 4 + KINDS.index(kind)) * 8 + rank,
                                               scale_range=_gain_matched_scales(K * tp if kind in ("o", "down") else K))
                self.layers.append(("layers.%d.%s" % (i, kind), kind, pt))
        h = shape.hidden
        dev = torch.device("cuda", torch.cuda.current_device())
        self.x = torch.zeros((batch, h), dtype=torch.bfloat16, device=dev)
        self.bufs = {}
        for name, kind, pt in self.layers[:4]:
            self.bufs[kind] = torch.zeros((batch, pt.N), dtype=torch.bfloat16, device=dev)
        self.x_host = torch.zeros((batch, h), dtype=torch.bfloat16, pin_memory=True)
        self.y_host = torch.zeros((batch, h), dtype=torch.bfloat16, pin_memory=True)
        self.stream = torch.cuda.Stream()
        need = max(pt.workspace_bytes(batch) for _, _, pt in self.layers)
        reserve_workspace(need, stream=self.stream)
        self.graph = None
        self.config: dict[str, int] = {}

    # ------------------------------------------------------------------
    @property
    def names(self) -> list[str]:
        return [n for n, _, _ in self.layers]

    def sizes(self) -> dict[str, int]:
        return {n: pt.N * pt.K for n, _, pt in self.layers}

    def weight_bytes(self) -> int:
        return sum(pt.nbytes for _, _, pt in self.layers)

    def step_bytes(self, config: dict[str, int]) -> int:
        """Algorithmic bytes of one decode step, this rank."""
        tot = 0
        for n, kind, pt in self.layers:
            r = config[n]
            tot += algorithmic_bytes(pt.N, pt.K, self.B, r, pt.planes_read(r), self.G)
        return tot

    def _all_reduce(self, t: torch.Tensor) -> None:
        if self.tp > 1:
            torch.distributed.all_reduce(t, group=self.pg)

    def _run(self, config: dict[str, int], pdl: bool = True) -> None:
        """One decode step on self.stream (launch-only; captured by capture())."""
        s = self.stream
        x = self.x
        b = self.bufs
        for name, kind, pt in self.layers:
            r = config[name]
            if kind == "qkv":
                pt.gemv(x, r, out=b["qkv"], pdl=pdl, stream=s)
            elif kind == "o":
                pt.gemv(b["qkv"][:, :pt.K], r, out=b["o"], pdl=pdl, stream=s)
                self._all_reduce(b["o"])
            elif kind == "gate_up":
                pt.gemv(b["o"], r, out=b["gate_up"], pdl=pdl, stream=s)
            else:
                pt.gemv(b["gate_up"][:, :pt.K], r, out=x, pdl=pdl, stream=s)
                self._all_reduce(x)

    def capture(self, config, pdl: bool = True) -> None:
        """(Re)capture the decode step for a per-layer bit-width config."""
        if isinstance(config, int):
            config = {n: config for n in self.names}
        missing = [n for n in self.names if n not in config]
        if missing:
            raise KeyError("incomplete config: missing %r" % missing[0])
        for r in config.values():
            if r not in LADDER:
                raise ValueError("bit-width %d not on the ladder" % r)
        self.config = dict(config)
        with torch.cuda.stream(self.stream):
            self._run(self.config, pdl)  # warm the launch path outside capture
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            self._run(self.config, pdl)
        self.graph = g

    def launches_per_step(self) -> int:
        return len(self.layers)

    def step(self) -> None:
        """Replay one captured decode step (device-resident activations)."""
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def decode(self, x_host: torch.Tensor | None = None) -> torch.Tensor:
        """End-to-end step through the public API: pinned host x -> device,
        replay, device y -> pinned host.  Returns the host tensor."""
        s = self.stream
        with torch.cuda.stream(s):
            src = self.x_host if x_host is None else x_host
            self.x.copy_(src, non_blocking=True)
            self.graph.replay()
            self.y_host.copy_(self.x, non_blocking=True)
        return self.y_host

    def io_bytes(self) -> tuple[int, int]:
        return self.x.numel() * 2, self.x.numel() * 2
