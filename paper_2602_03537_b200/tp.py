"""Tensor-parallel sharding of sliced linears (BASELINE config C5).

One process per GPU.  A parent (codes (N, K) uint8 + scales (N, ceil(K/G)))
is sharded once at load time; every rank slices its shard in place to the
layer's r (identical on every rank), so no repacking is ever needed:

* column-parallel (qkv, gate_up): rows split -- rank j owns rows
  [n0, n1); outputs are disjoint, no exchange;
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
    rows: tuple[int, int]
    cols: tuple[int, int]
    groups: tuple[int, int]

    @property
    def shape(self) -> tuple[int, int]:
        return self.rows[1] - self.rows[0], self.cols[1] - self.cols[0]


def shard_plan(kind: str, N: int, K: int, tp: int, rank: int, group_size: int = 128,
               row_quantum: int = 16) -> Shard:
    """The slice of an (N, K) parent that ``rank`` of ``tp`` owns."""
    if not 0 <= rank < tp:
        raise ValueError("rank %d outside [0, %d)" % (rank, tp))
    ng = -(-K // group_size)
    if kind in COLUMN:
        r0, r1 = _even_split(N, tp, rank, row_quantum)
        return Shard(kind, "column", (r0, r1), (0, K), (0, ng))
    if kind in ROW:
        g0, g1 = _even_split(ng, tp, rank)
        return Shard(kind, "row", (0, N), (g0 * group_size, min(K, g1 * group_size)), (g0, g1))
    raise KeyError(kind)


def shard_parent(codes: np.ndarray, scales: np.ndarray, plan: Shard):
    """(codes, scales) of one shard, contiguous."""
    r0, r1 = plan.rows
    k0, k1 = plan.cols
    g0, g1 = plan.groups
    return (np.ascontiguousarray(codes[r0:r1, k0:k1]), np.ascontiguousarray(scales[r0:r1, g0:g1]))


def shard_activations(X, plan: Shard):
    """The K slice of the activations a row-parallel shard consumes."""
    k0, k1 = plan.cols
    return X[:, k0:k1] if plan.parallel == "row" else X


class TPLinear:
    """One rank's shard of a sliced linear; forward = K3/K4 (+ all-reduce for row-parallel)."""

    def __init__(self, codes: np.ndarray, scales: np.ndarray, kind: str, tp: int, rank: int,
                 group_size: int = 128, process_group=None):
        from .device import PlaneTensor

        self.plan = shard_plan(kind, codes.shape[0], codes.shape[1], tp, rank, group_size)
        c, s = shard_parent(codes, scales, self.plan)
        self.planes = PlaneTensor.from_codes(c, 8, s, group_size)
        self.tp, self.pg = tp, process_group

    def __call__(self, X, r: int, out=None):
        import torch.distributed as dist

        y = self.planes.linear(shard_activations(X, self.plan), r, out=out)
        if self.plan.parallel == "row" and self.tp > 1:
            dist.all_reduce(y, group=self.pg)
        return y
