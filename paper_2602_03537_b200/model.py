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

import torch

from . import _lib
from .device import LADDER, PlaneTensor, algorithmic_bytes, reserve_workspace
from .shapes import (KINDS, KINDS_UNFUSED, LLAMA31_8B, PHI3_MEDIUM, QWEN3_14B, SHAPES,  # noqa: F401
                     DecoderShape, full_layer_dims, layer_names)


def tp_layer_dims(shape: DecoderShape, kind: str, tp: int, rank: int = 0) -> tuple[int, int]:
    """(N, K) of rank ``rank``'s shard (tp.decoder_plan: q heads + their kv
    heads / gate + up rows for column-parallel, whole scale groups of K for
    row-parallel)."""
    if tp == 1:
        return full_layer_dims(shape, kind)
    from .tp import decoder_plan

    return decoder_plan(shape, kind, tp, rank).shape


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
                 n_layers: int | None = None, fused: bool = True, shard_from_full: bool = False):
        _lib.require_cuda()
        if batch < 1 or batch > 32:
            raise ValueError("decode batch must lie in [1, 32]")
        self.shape = shape
        self.B = batch
        self.G = group_size
        self.tp, self.rank, self.pg = tp, rank, process_group
        self.n_layers = n_layers or shape.n_layers
        self.fused = fused
        kinds = KINDS if fused else KINDS_UNFUSED
        self.layers: list[tuple[str, str, PlaneTensor]] = []
        # (seed, scale_range, signed_rows) of each layer's synthetic parent: PlaneTensor.random_parent
        # regenerates the same codes and scales from them (the parity tests do)
        self.parent_seeds: list[tuple[int, tuple[float, float]]] = []
        for i in range(self.n_layers):
            for kind in kinds:
                N, K = tp_layer_dims(shape, kind, tp, rank)
                sr = _gain_matched_scales(K * tp if kind in ("o", "down") else K)
                if shard_from_full and tp > 1:
                    # this rank's shard (tp.decoder_plan) of the parent a tp = 1 stack with the
                    # same seed holds: the TP step must reproduce the single-GPU step
                    from .tp import decoder_plan

                    sd = seed * 1000003 + (i * 8 + kinds.index(kind)) * 8
                    fN, fK = full_layer_dims(shape, kind)
                    codes, scales = PlaneTensor.random_parent_codes(fN, fK, group_size, sd,
                                                                    _gain_matched_scales(fK), True)
                    plan = decoder_plan(shape, kind, tp, rank, group_size)
                    rows = torch.cat([torch.arange(a, b, device=codes.device) for a, b in plan.segments])
                    (k0, k1), (g0, g1) = plan.cols, plan.groups
                    pt = PlaneTensor.from_codes(codes[rows, k0:k1].contiguous(), 8,
                                                scales[rows, g0:g1].contiguous(), group_size)
                    del codes, scales
                else:
                    sd = seed * 1000003 + (i * 8 + kinds.index(kind)) * 8 + rank
                    pt = PlaneTensor.random_parent(N, K, group_size, seed=sd, scale_range=sr, signed_rows=True)
                self.layers.append(("layers.%d.%s" % (i, kind), kind, pt))
                self.parent_seeds.append((sd, sr, True))
        self.stream = torch.cuda.Stream()
        self.set_batch(batch)
        self.graph = None
        self.program = None
        self.config: dict[str, int] = {}

    def set_batch(self, batch: int) -> None:
        """(Re)allocate the activation buffers for decode batch ``batch``; the
        resident weights are untouched.  Drops any captured step."""
        if batch < 1 or batch > 32:
            raise ValueError("decode batch must lie in [1, 32]")
        self.B = batch
        kinds = KINDS if self.fused else KINDS_UNFUSED
        h = self.shape.hidden
        dev = torch.device("cuda", torch.cuda.current_device())
        self.graph = None
        self.program = None
        self.programs = []
        self.x = torch.zeros((batch, h), dtype=torch.bfloat16, device=dev)
        self.bufs = {}
        for name, kind, pt in self.layers[:len(kinds)]:
            self.bufs[kind] = torch.zeros((batch, pt.N), dtype=torch.bfloat16, device=dev)
        self.x_host = torch.zeros((batch, h), dtype=torch.bfloat16, pin_memory=True)
        self.y_host = torch.zeros((batch, h), dtype=torch.bfloat16, pin_memory=True)
        need = max(pt.workspace_bytes(batch) for _, _, pt in self.layers)
        reserve_workspace(need, stream=self.stream)

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
        # fused: x -> qkv -> (q part) -> o -> gate_up -> (gate part) -> down -> x
        # unfused: x -> q, k, v; q -> o; o -> gate, up; gate -> down -> x
        src = {"qkv": lambda pt: x, "q": lambda pt: x, "k": lambda pt: x, "v": lambda pt: x,
               "o": lambda pt: (b["qkv"][:, :pt.K] if self.fused else b["q"]),
               "gate_up": lambda pt: b["o"], "gate": lambda pt: b["o"], "up": lambda pt: b["o"],
               "down": lambda pt: (b["gate_up"][:, :pt.K] if self.fused else b["gate"])}
        for name, kind, pt in self.layers:
            r = config[name]
            out = x if kind == "down" else b[kind]
            pt.linear(src[kind](pt), r, out=out, pdl=pdl, stream=s)
            if kind in ("o", "down"):
                self._all_reduce(out)

    def _stack_layers(self):
        """(PlaneTensor, X, Y) per layer in order, the same dataflow as _run."""
        b, x = self.bufs, self.x
        out = []
        for name, kind, pt in self.layers:
            if kind in ("qkv", "q", "k", "v"):
                X = x
            elif kind == "o":
                X = b["qkv"][:, :pt.K] if self.fused else b["q"]
            elif kind in ("gate_up", "gate", "up"):
                X = b["o"]
            else:
                X = b["gate_up"][:, :pt.K] if self.fused else b["gate"]
            out.append((pt, X, x if kind == "down" else b[kind]))
        return out

    def stack_kernel_ok(self, config) -> bool:
        """Where the persistent K3S path is the default (single GPU, B <= 16,
        G = 128), from scripts/stack_matrix.py (profiles/r1_stack_matrix*.txt):
        * uniform r: see the table in the body (profiles/r2_dispatch_matrix.txt);
        * heterogeneous (per-layer r, parents): at B <= 2, fused or unfused.
        stack_kernel=True / False forces either path."""
        rs = set(config.values()) if isinstance(config, dict) else {int(config)}
        parents = all(pt.nplanes == 8 for _, _, pt in self.layers)
        if len(rs) == 1:
            # measured (scripts/dispatch_matrix.py, profiles/r2_dispatch_matrix.txt): K3S wins
            # at B <= 8 for every r and up to B = 16 for r != 8
            r0 = next(iter(rs))
            ok = self.B <= 8 or r0 != 8
        else:
            # per-layer r (the dispatch kernel): 1.61 vs 1.96 ms fused, 2.02 vs 2.16 ms for the
            # 224 unfused linears of C3 at B = 1, 2.15 vs 2.18 at B = 2; from B = 3 the graph
            # wins (2.21 vs 2.94 ms; scripts/hetero_matrix.py, profiles/r2_hetero_matrix.txt)
            ok = parents and self.B <= 2
        return ok and self.B <= 16 and self.G == 128  # tp > 1: one K3S launch per all-reduce segment

    def capture(self, config, pdl: bool = True, stack_kernel: bool | None = None, graph: bool = True) -> None:
        """(Re)capture the decode step for a per-layer bit-width config.

        Single-GPU stacks with B <= 16 run as ONE persistent K3S launch per step
        (weights keep streaming across layer boundaries; a heterogeneous config
        dispatches per layer inside the kernel); under TP one K3S launch per
        segment between all-reduces; otherwise a CUDA graph of per-layer K3
        launches with PDL."""
        if isinstance(config, int):
            config = {n: config for n in self.names}
        missing = [n for n in self.names if n not in config]
        if missing:
            raise KeyError("incomplete config: missing %r" % missing[0])
        for r in config.values():
            if r not in LADDER:
                raise ValueError("bit-width %d not on the ladder" % r)
        self.config = dict(config)
        use_stack = self.stack_kernel_ok(self.config) if stack_kernel is None else stack_kernel
        self.program = None
        self.programs = []
        if use_stack and self.tp > 1:
            # TP: one persistent K3S launch per segment between all-reduces
            # (x -> qkv -> o | all-reduce | -> gate_up -> down | all-reduce), the
            # segment's last layer being the row-parallel one whose partial is summed
            from .device import StackProgram

            sl = self._stack_layers()
            seg = []
            for (name, kind, _), lay in zip(self.layers, sl):
                seg.append((name, lay))
                if kind in ("o", "down"):
                    rs = [self.config[n] for n, _ in seg]
                    self.programs.append((StackProgram([l for _, l in seg], rs[0] if len(set(rs)) == 1 else rs,
                                                       self.B), lay[2]))
                    seg = []

            def run():
                for prog, out in self.programs:
                    prog.run(self.stream)
                    self._all_reduce(out)
        elif use_stack:
            from .device import StackProgram

            rs = [self.config[n] for n, _, _ in self.layers]
            self.program = StackProgram(self._stack_layers(), rs[0] if len(set(rs)) == 1 else rs, self.B)
            run = lambda: self.program.run(self.stream)  # noqa: E731
        else:
            run = lambda: self._run(self.config, pdl)  # noqa: E731
        # buffers (and any activations the caller wrote) were produced on the caller's stream
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            run()  # warm the launch path outside capture
        self.stream.synchronize()
        self._eager = run
        if not graph:  # e.g. a gloo process group: its collectives cannot be graph-captured
            self.graph = None
            return
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            run()
        self.graph = g

    def launches_per_step(self) -> int:
        """libmatq kernel launches per step (NCCL's all-reduce kernels not counted)."""
        if getattr(self, "programs", None):
            return len(self.programs)
        return 1 if getattr(self, "program", None) is not None else len(self.layers)

    def step(self) -> None:
        """Replay one captured decode step (device-resident activations)."""
        self.stream.wait_stream(torch.cuda.current_stream())  # activations written by the caller
        with torch.cuda.stream(self.stream):
            if self.graph is None:
                self._eager()
            else:
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
