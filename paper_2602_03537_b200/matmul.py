"""Matmul over bit-plane weights with in-register dequantisation.

Drop-in for /root/reference/pkg/src/nestquant/matmul.py.  Same names,
validation and messages; the compute runs on the B200 through libmatq:

* ``matmul_packed``  -> mq_gemv (K3): bitsliced slice + exact bf16 decode +
  mma.m16n8k16 with fp32 accumulation per scale group.  The reference takes
  fp32 activations (matmul.py:72-82); K3 splits each fp32 activation into
  bf16 hi + lo terms on device so the product keeps ~16 mantissa bits
  (max rel err ~1e-6 vs matmul_ref, inside the reference's 1e-4 gate,
  test_matmul.py:19-20).
* ``matmul_ref``     -> mq_dequant + mq_matmul_ref: the oracle arithmetic,
  float32 k-ascending, bit-identical to the reference's numpy loop.

Bit-widths: the reference's PackedLayer accepts r in {2, 3, 4}
(matmul.py:55-56); here any r on the ladder {2, 3, 4, 6, 8} works, and
``PackedLayer.from_parent`` serves every r from one resident int8 parent
without repacking (mode P).
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, kernels
from .device import LADDER, PlaneTensor
from .packing import PackedTensor, _padded_cols, pack, to_canonical, unpack_device
from .slicing import NestedLayer, SlicedLayer


class MatmulError(ValueError):
    pass


@dataclass
class PackedLayer:
    """Inference-ready layer: r-bit codes in device bit planes + effective scales.

    matmul.py:29-69.  ``packed`` is the reference-format PackedTensor when the
    layer was built from one (r in {2,3,4}); ``device()`` is the P8 plane
    tensor the GEMV reads.
    """

    name: str
    packed: PackedTensor | None
    scales: np.ndarray  # float32, (d_row, n_groups) effective scales
    group_size: int
    _bits: int | None = None
    _shape: tuple[int, int] | None = None
    _planes: PlaneTensor | None = field(default=None, repr=False)
    _parent_r: int | None = None

    def __post_init__(self):
        self.scales = np.ascontiguousarray(self.scales, dtype=np.float32)
        if self.packed is not None:
            self._bits = self.packed.bits
            self._shape = tuple(self.packed.shape)
        self._planes_key = None

    @property
    def bits(self) -> int:
        return self._bits

    @property
    def zero_code(self) -> int:
        return 1 << (self.bits - 1)

    @property
    def shape(self) -> tuple[int, int]:
        return self._shape

    @classmethod
    def from_sliced(cls, layer: SlicedLayer) -> "PackedLayer":
        """matmul.py:53-62; r in {6, 8} is accepted as well (no reference format)."""
        if layer.bits not in LADDER:
            raise MatmulError("unsupported bits")
        packed = pack(layer.codes, layer.bits) if layer.bits <= 4 else None
        out = cls(name=layer.name, packed=packed, scales=layer.scales, group_size=layer.group_size,
                  _bits=layer.bits, _shape=tuple(layer.codes.shape))
        if packed is None:
            out._planes = PlaneTensor.from_codes(layer.codes, layer.bits, layer.scales,
                                                 layer.group_size, scales_are_effective=True)
        return out

    @classmethod
    def from_parent(cls, parent: NestedLayer | PlaneTensor, r: int, name: str | None = None
                    ) -> "PackedLayer":
        """Mode P: an r-bit view on the resident parent planes (no repacking)."""
        if r not in LADDER:
            raise MatmulError("unsupported bits")
        pt = parent.device() if isinstance(parent, NestedLayer) else parent
        scales = np.zeros((0, 0), np.float32)
        out = cls(name=name or getattr(parent, "name", "parent"), packed=None, scales=scales,
                  group_size=pt.G, _bits=r, _shape=pt.shape, _planes=pt, _parent_r=r)
        return out

    def device(self) -> PlaneTensor:
        """The P8 planes the GEMV reads (built on first use, cached)."""
        if self._planes is not None and self._parent_r is not None:
            return self._planes
        key = (id(self.packed), self.scales.ctypes.data, self.group_size)
        if self._planes is None or (self.packed is not None and self._planes_key != key):
            if self.packed is None:
                raise MatmulError("layer has no packed codes")
            codes = unpack_device(to_canonical(self.packed))
            self._planes = PlaneTensor.from_codes(codes, self.bits, self.scales, self.group_size,
                                                  scales_are_effective=True)
            self._planes_key = key
        return self._planes

    def dense_f32(self) -> np.ndarray:
        """(codes - z) * scales[:, col // G] in float32 (matmul.py:64-69), on device."""
        return self.device().decode(self.bits).cpu().numpy()


@dataclass
class MatmulTask:
    """matmul.py:72-82."""

    X: np.ndarray  # float32, (batch, d_col)
    layer: PackedLayer

    def __post_init__(self):
        self.X = np.ascontiguousarray(self.X, dtype=np.float32)
        if self.X.ndim != 2:
            raise MatmulError("activations must be (batch, d_col)")
        if self.X.shape[1] != self.layer.shape[1]:
            raise MatmulError("shape mismatch")


def matmul_ref(task: MatmulTask) -> np.ndarray:
    """Dense reference: float32, k-ascending (matmul.py:85-92); exact on device."""
    _lib.require_cuda()
    W = task.layer.device().decode(task.layer.bits)
    X = torch.from_numpy(task.X).cuda()
    B, K = task.X.shape
    N = W.shape[0]
    Y = torch.empty((B, N), dtype=torch.float32, device="cuda")
    _lib.call("mq_matmul_ref", _lib.ptr(X), B, K, _lib.ptr(W), N, _lib.ptr(Y), _lib.stream_ptr())
    return Y.cpu().numpy()


def _validate(layer: PackedLayer) -> None:
    if layer.bits not in LADDER:
        raise MatmulError("unsupported bits")
    if layer.group_size % 32 != 0:
        raise MatmulError("group size must be a multiple of 32")


def matmul_packed_device(layer: PackedLayer, X: torch.Tensor, out: torch.Tensor | None = None,
                         out_dtype: torch.dtype | None = None) -> torch.Tensor:
    """Device-in / device-out packed matmul: K3 for B <= 32, K4 (tcgen05) for
    larger bf16 batches, K3 in chunks for fp32 activations."""
    _validate(layer)
    return layer.device().linear(X, layer.bits, out=out, out_dtype=out_dtype)


def matmul_packed(task: MatmulTask, force_fallback: bool = False) -> np.ndarray:
    """Packed matmul on the B200 (matmul.py:103-120).

    ``force_fallback`` is accepted for signature compatibility only: there is
    no fallback backend, both values run the sm_100a kernel.
    """
    layer = task.layer
    _validate(layer)
    _lib.require_cuda()
    X = torch.from_numpy(task.X).cuda()
    Y = matmul_packed_device(layer, X, out_dtype=torch.float32)
    return Y.cpu().numpy()


def random_task(m: int, k: int, batch: int, bits: int, group_size: int = 128,
                seed: int = 0) -> MatmulTask:
    """Seeded random packed layer + activations (matmul.py:123-135; same RNG stream)."""
    if bits not in LADDER:
        raise MatmulError("unsupported bits")
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 1 << bits, size=(m, k), dtype=np.int64)
    n_groups = -(-k // group_size)
    scales = rng.uniform(0.005, 0.02, size=(m, n_groups)).astype(np.float32)
    if bits <= 4:
        layer = PackedLayer(name="bench", packed=pack(codes, bits), scales=scales,
                            group_size=group_size)
    else:
        from .slicing import SlicedLayer

        layer = PackedLayer.from_sliced(SlicedLayer("bench", bits, codes.astype(np.uint8), scales,
                                                    group_size, bits))
    X = rng.standard_normal((batch, k)).astype(np.float32)
    return MatmulTask(X=X, layer=layer)


def _time_ns(fn, reps: int) -> tuple[int, list[int]]:
    """Warm-up + median of reps (matmul.py:138-145), timed with CUDA events."""
    fn()
    torch.cuda.synchronize()
    samples = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        samples.append(int(e0.elapsed_time(e1) * 1e6))
    return int(statistics.median(samples)), samples


def bench(m: int, k: int, batch: int, bits: int, reps: int = 7, group_size: int = 128,
          seed: int = 0) -> list[dict]:
    """Time the packed GEMV against a dense bf16 cuBLAS matmul (matmul.py:148-192).

    Same record keys as the reference.  Activations and outputs stay on the
    device (bf16); ``gbps`` counts the weight payload + X + Y like the
    reference (matmul.py:167-168, scales excluded).
    """
    if reps < 3:
        raise MatmulError("reps must be >= 3")
    if bits not in LADDER:
        raise MatmulError("unsupported bits")
    task = random_task(m, k, batch, bits, group_size=group_size, seed=seed)
    pt = task.layer.device()
    X = torch.from_numpy(task.X).cuda().to(torch.bfloat16)
    Wd = pt.decode(bits).to(torch.bfloat16)
    dense_ns, _ = _time_ns(lambda: X @ Wd.T, reps)
    out = torch.empty((batch, m), dtype=torch.bfloat16, device="cuda")
    weight_bytes = (task.layer.packed.payload_bytes if task.layer.packed is not None
                    else bits * m * _padded_cols(k) // 8)
    bytes_moved = weight_bytes + 2 * batch * k + 2 * batch * m
    median_ns, samples = _time_ns(
        lambda: matmul_packed_device(task.layer, X, out=out), reps)
    return [{
        "m": m, "k": k, "batch": batch, "bits": bits,
        "median_ns": median_ns,
        "gbps": bytes_moved / median_ns if median_ns else 0.0,
        "speedup": dense_ns / median_ns if median_ns else 0.0,
        "backend": kernels.backend_name(),
        "weight_bytes": weight_bytes,
        "bytes_moved": bytes_moved,
        "dense_median_ns": dense_ns,
        "samples_ns": samples,
    }]
