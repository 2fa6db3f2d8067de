"""``MatLinear``: the quantized-linear torch module of the hot path.

The reference has no nn.Module: its "quantized linear" is a ``PackedLayer``
driven by ``matmul_packed`` (matmul.py:29-69, :103-120).  ``MatLinear`` wraps
one resident int8 parent (P8 blob) and slices it to ``bits`` on the fly:

* decode batches (<= 16 rows)  -> K3, the sliced GEMV (mma.sync, bitsliced decode)
* prefill batches (> 16 rows) -> K4, the tcgen05 dequant-GEMM

``bits`` can be changed at any time (``set_bits``) without touching the weights
-- the per-layer bit-width of an EvoPress-style config is just an attribute.
Inputs of any leading shape (..., in_features) in bf16 (fp32 is accepted and
goes through K3 with the hi/lo split); output bf16 (or fp32 for fp32 input).
There is no backward: the parent is a frozen inference artefact.
"""

from __future__ import annotations

import torch

from .device import LADDER, PlaneTensor

__all__ = ["MatLinear"]


class MatLinear(torch.nn.Module):
    def __init__(self, planes: PlaneTensor, bits: int = 4, bias: torch.Tensor | None = None,
                 name: str = ""):
        super().__init__()
        if bits not in LADDER:
            raise ValueError("unsupported bits")
        planes._check(bits)
        self.planes = planes
        self.bits = int(bits)
        self.name = name
        self.in_features, self.out_features = planes.K, planes.N
        if bias is not None:
            bias = bias.detach().to(device="cuda", dtype=torch.float32).contiguous()
            if bias.shape != (planes.N,):
                raise ValueError("bias must be (out_features,)")
        self.register_buffer("bias", bias, persistent=False)

    # -- construction ----------------------------------------------------
    @classmethod
    def from_codes(cls, codes, scales, group_size: int = 128, bits: int = 4, bias=None, name: str = ""):
        """int8 parent codes (out, in) + fp32 group scales (out, ceil(in/G))."""
        return cls(PlaneTensor.from_codes(codes, 8, scales, group_size), bits, bias, name)

    @classmethod
    def from_nested(cls, layer, bits: int = 4, bias=None) -> "MatLinear":
        """From a reference-style ``NestedLayer`` (slicing.py:57-91)."""
        return cls(layer.device(), bits, bias, getattr(layer, "name", ""))

    def set_bits(self, bits: int) -> "MatLinear":
        if bits not in LADDER:
            raise ValueError("unsupported bits")
        self.planes._check(bits)
        self.bits = int(bits)
        return self

    # -- forward ---------------------------------------------------------
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.shape[-1] != self.in_features:
            raise ValueError("expected (..., %d) activations" % self.in_features)
        lead = x.shape[:-1]
        x2 = x.reshape(-1, self.in_features)
        if x2.dtype not in (torch.bfloat16, torch.float32):
            x2 = x2.to(torch.bfloat16)
        if not x2.is_cuda:
            raise ValueError("activations must be CUDA tensors")
        y = self.planes.linear(x2, self.bits)
        if self.bias is not None:
            y = (y.float() + self.bias).to(y.dtype)
        return y.reshape(*lead, self.out_features)

    def dequantized_weight(self) -> torch.Tensor:
        """fp32 (out, in) weights at the current bit-width (bit-exact dense_f32)."""
        return self.planes.decode(self.bits)

    def extra_repr(self) -> str:
        return "in_features=%d, out_features=%d, bits=%d (int8 parent, G=%d)" % (
            self.in_features, self.out_features, self.bits, self.planes.G)

    @staticmethod
    def random(out_features: int, in_features: int, bits: int = 4, seed: int = 0) -> "MatLinear":
        return MatLinear(PlaneTensor.random_parent(out_features, in_features, seed=seed), bits)


