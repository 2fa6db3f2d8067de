"""Tensor-parallel sharding of sliced linears (BASELINE config C5).

One process per GPU.  A parent (codes (N, K) uint8 + scales (N, ceil(K/G)))
is sharded once at load time; every rank slices its shard in place to the
layer's r (identical on every rank), so no repacking is ever needed:

* column-parallel (qkv, gate_up): rows split per constituent -- rank j owns
  its q heads and their k / v heads, and gate rows [i0, i1) with the same up
  rows (``decoder_plan``); outputs are disjoint, no exchange;
* row-parallel (o, down): K split on scale-group boundaries -- rank j owns
  columns [k0, k1) and the matching scale groups; partial outputs are summed
  with one all-reduce of the (B, N) activation.

K is split in whole groups so that no scale group straddles two ranks.  When
the group count does not divide evenly (Phi-3-Medium down at TP=8: 140
groups / 8 = 17.5) the first ``ngroups % tp`` ranks take one extra group
(SURVEY 7.4 item 7).

The host-side math here is exercised on CPU with the gloo backend
(tests/test_tp.py, world size 2); on GPUs the same plan feeds
``TPLinear`` over NCCL.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

COLUMN = ("qkv", "gate_up", "q", "k", "v", "gate", "up")
ROW = ("o", "down")


def _even_split(total: int, parts: int, rank: int, quantum: int = 1) -> tuple[int, int]:
    """[lo, hi) of ``rank`` when ``total`` units of ``quantum`` are dealt
    as evenly as possible (the first ``n % parts`` ranks get one more)."""
    units = -(-total // quantum)
    base, extra = divmod(units, parts)
    lo_u = rank * base + min(rank, extra)
    hi_u = lo_u + base + (1 if rank < extra else 0)
    return min(total, lo_u * quantum), min(total, hi_u * quantum)


@dataclass(frozen=True)
class Shard:
    kind: str
    parallel: str  # "column" | "row"
    segments: tuple[tuple[int, int], ...]  # parent row ranges this rank owns, in order
    cols: tuple[int, int]
    groups: tuple[int, int]

    @property
    def rows(self) -> tuple[int, int]:
        """[lo, hi) of a single-segment shard (row-parallel and unfused column shards)."""
        if len(self.segments) != 1:
            raise ValueError("a fused shard owns %d row segments" % len(self.segments))
        return self.segments[0]

    @property
    def shape(self) -> tuple[int, int]:
        return sum(b - a for a, b in self.segments), self.cols[1] - self.cols[0]


def shard_plan(kind: str, N: int, K: int, tp: int, rank: int, group_size: int = 128,
               row_quantum: int = 16, parts=None) -> Shard:
    """The slice of an (N, K) parent that ``rank`` of ``tp`` owns.

    ``parts``: for a FUSED column-parallel linear, its constituents in row
    order as (rows, quantum) pairs -- e.g. gate_up = ((inter, 16), (inter, 16)),
    qkv = ((q, head_dim), (kv, head_dim), (kv, head_dim)).  Each constituent is
    split on its own, so rank j owns gate rows [i0, i1) AND the matching up
    rows, and its SiLU(gate) * up feeds its own K shard of down; without
    ``parts`` a column shard is one contiguous row range."""
    if not 0 <= rank < tp:
        raise ValueError("rank %d outside [0, %d)" % (rank, tp))
    ng = -(-K // group_size)
    if kind in COLUMN:
        if parts is None:
            parts = ((N, row_quantum),)
        if sum(p[0] for p in parts) != N:
            raise ValueError("constituents of %s cover %d rows, not %d" % (kind, sum(p[0] for p in parts), N))
        segs, base = [], 0
        for size, quantum in parts:
            lo, hi = _even_split(size, tp, rank, quantum)
            segs.append((base + lo, base + hi))
            base += size
        return Shard(kind, "column", tuple(segs), (0, K), (0, ng))
    if kind in ROW:
        g0, g1 = _even_split(ng, tp, rank)
        return Shard(kind, "row", ((0, N),), (g0 * group_size, min(K, g1 * group_size)), (g0, g1))
    raise KeyError(kind)


def decoder_plan(shape, kind: str, tp: int, rank: int, group_size: int = 128) -> Shard:
    """Shard of one linear of a decoder (shapes.DecoderShape) for Megatron-style
    TP: q heads and the intermediate range split per rank; k / v heads split
    when tp divides them, else each rank holds (replicated) exactly the kv heads
    its q heads attend to (GQA group = n_heads / n_kv_heads; SURVEY 7.4 item 7,
    Phi-3-Medium: 10 kv heads at tp 4 / 8)."""
    from .shapes import full_layer_dims

    N, K = full_layer_dims(shape, kind)
    hd = shape.head_dim
    if kind == "gate_up":
        # whole scale groups, so the range equals this rank's K shard of down
        return shard_plan(kind, N, K, tp, rank, group_size,
                          parts=((shape.intermediate, group_size), (shape.intermediate, group_size)))
    if kind in ("qkv", "k", "v"):
        q0, q1 = _even_split(shape.n_heads, tp, rank)
        if shape.n_kv_heads % tp == 0:
            k0, k1 = _even_split(shape.n_kv_heads, tp, rank)
        else:  # replicate: the kv heads of this rank's q heads
            grp = shape.n_heads // shape.n_kv_heads
            k0, k1 = (q0 // grp, (q1 - 1) // grp + 1) if q1 > q0 else (0, 0)
        kv = shape.kv_out
        if kind == "qkv":
            segs = ((q0 * hd, q1 * hd), (shape.q_out + k0 * hd, shape.q_out + k1 * hd),
                    (shape.q_out + kv + k0 * hd, shape.q_out + kv + k1 * hd))
        else:
            segs = ((k0 * hd, k1 * hd),)
        return Shard(kind, "column", segs, (0, K), (0, -(-K // group_size)))
    if kind == "q":
        q0, q1 = _even_split(shape.n_heads, tp, rank)
        return Shard(kind, "column", ((q0 * hd, q1 * hd),), (0, K), (0, -(-K // group_size)))
    if kind in ("gate", "up"):
        return shard_plan(kind, N, K, tp, rank, group_size, row_quantum=group_size)
    return shard_plan(kind, N, K, tp, rank, group_size)  # o / down: K on whole scale groups


def shard_parent(codes: np.ndarray, scales: np.ndarray, plan: Shard):
    """(codes, scales) of one shard, contiguous (a fused shard's row segments
    concatenated in order)."""
    k0, k1 = plan.cols
    g0, g1 = plan.groups
    rows = np.concatenate([np.arange(a, b) for a, b in plan.segments]) if plan.segments else np.zeros(0, int)
    return (np.ascontiguousarray(codes[rows, k0:k1]), np.ascontiguousarray(scales[rows, g0:g1]))


def shard_activations(X, plan: Shard):
    """The K slice of the activations a row-parallel shard consumes."""
    k0, k1 = plan.cols
    return X[:, k0:k1] if plan.parallel == "row" else X


class TPLinear:
    """One rank's shard of a sliced linear; forward = K3/K4 (+ all-reduce for row-parallel)."""

    def __init__(self, codes: np.ndarray, scales: np.ndarray, kind: str, tp: int, rank: int,
                 group_size: int = 128, process_group=None, plan: Shard | None = None):
        from .device import PlaneTensor

        self.plan = plan or shard_plan(kind, codes.shape[0], codes.shape[1], tp, rank, group_size)
        c, s = shard_parent(codes, scales, self.plan)
        self.planes = PlaneTensor.from_codes(c, 8, s, group_size)
        self.tp, self.pg = tp, process_group

    def __call__(self, X, r: int, out=None):
        import torch.distributed as dist

        y = self.planes.linear(shard_activations(X, self.plan), r, out=out)
        if self.plan.parallel == "row" and self.tp > 1:
            dist.all_reduce(y, group=self.pg)
        return y
