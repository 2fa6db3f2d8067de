"""Decoder shapes of the BASELINE configs (pure Python: no torch, no libmatq).

bench.py's reference arm loads this file by path, so the CPU reference run
shares the workload definition without importing the package (which maps
libmatq.so).  Model shapes come from the public model configs; the reference
names the models only.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class DecoderShape:
    name: str
    hidden: int
    intermediate: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    n_layers: int
    qk_norm: bool = False  # per-head RMSNorm of q and k before the rotary embedding (Qwen3)

    @property
    def qkv_out(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def q_out(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_out(self) -> int:
        return self.n_kv_heads * self.head_dim


LLAMA31_8B = DecoderShape("Llama-3.1-8B", 4096, 14336, 32, 8, 128, 32)
QWEN3_14B = DecoderShape("Qwen3-14B", 5120, 17408, 40, 8, 128, 40, qk_norm=True)
PHI3_MEDIUM = DecoderShape("Phi-3-Medium", 5120, 17920, 40, 10, 128, 40)
SHAPES = {s.name: s for s in (LLAMA31_8B, QWEN3_14B, PHI3_MEDIUM)}

KINDS = ("qkv", "o", "gate_up", "down")
# unfused linears (heterogeneous configs assign r per q / k / v / gate / up, BASELINE C3)
KINDS_UNFUSED = ("q", "k", "v", "o", "gate", "up", "down")


def layer_names(shape: DecoderShape, fused: bool = True) -> list[str]:
    kinds = KINDS if fused else KINDS_UNFUSED
    return ["layers.%d.%s" % (i, k) for i in range(shape.n_layers) for k in kinds]


def full_layer_dims(shape: DecoderShape, kind: str) -> tuple[int, int]:
    """(N, K) of an unsharded linear (fused qkv / gate_up, or unfused)."""
    h, inter, hd = shape.hidden, shape.intermediate, shape.head_dim
    dims = {"qkv": (shape.qkv_out, h), "o": (h, shape.q_out), "gate_up": (2 * inter, h),
            "down": (h, inter), "q": (shape.q_out, h), "k": (shape.n_kv_heads * hd, h),
            "v": (shape.n_kv_heads * hd, h), "gate": (inter, h), "up": (inter, h)}
    return dims[kind]
