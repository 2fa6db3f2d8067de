"""Device-resident bit-plane weights (the P8 layout) and the GEMV entry.

A ``PlaneTensor`` owns the MSB-first bit planes of one (N, K) layer in HBM
plus its tiled fp32 group scales.  A parent (``nbits = c``,
normally the int8 parent with c = 8) serves every slice r <= c without
repacking: slice r reads planes 0..r (mode P).  A child (``nbits = r``)
holds an already-sliced r-bit code (mode C) and streams exactly r/8 of the
parent's bytes.

Everything here is a thin shell over libmatq (include/matq.h); there is no
CPU compute path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

LADDER = (2, 3, 4, 6, 8)
MAX_GEMV_ROWS = 32


def _as_device_u8(codes) -> torch.Tensor:
    if isinstance(codes, torch.Tensor):
        t = codes
        if t.dtype != torch.uint8:
            t = t.to(torch.uint8)
        return t.cuda().contiguous()
    return torch.from_numpy(np.ascontiguousarray(codes, dtype=np.uint8)).cuda()


def _as_device_f32(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


class _Workspaces:
    """Per (device, stream) zero-initialised GEMV split-K workspaces."""

    def __init__(self):
        self._bufs: dict[tuple[int, int], torch.Tensor] = {}

    def get(self, nbytes: int, stream_ptr: int) -> torch.Tensor | None:
        if nbytes == 0:
            return None
        key = (torch.cuda.current_device(), stream_ptr)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError("matq workspace must be reserved before CUDA graph capture "
                                   "(call reserve_workspace)")
            size = max(nbytes, 1 << 20)
            buf = torch.zeros(size, dtype=torch.uint8, device="cuda")
            self._bufs[key] = buf
        return buf


WORKSPACES = _Workspaces()


def reserve_workspace(nbytes: int, stream=None) -> None:
    WORKSPACES.get(int(nbytes), _lib.stream_ptr(stream))


class PlaneTensor:
    """Bit planes + tiled scales of one layer on the current CUDA device."""

    def __init__(self, planes: torch.Tensor, tscales: torch.Tensor, N: int, K: int, G: int,
                 nbits: int, is_child: bool, scales_are_effective: bool):
        self.planes = planes
        self.tscales = tscales
        self.N, self.K, self.G = int(N), int(K), int(G)
        self.nbits = int(nbits)
        self.is_child = bool(is_child)
        self.scales_are_effective = bool(scales_are_effective)

    # -- construction ------------------------------------------------------
    @classmethod
    def from_codes(cls, codes, nbits: int, scales, group_size: int, is_child: bool = False,
                   scales_are_effective: bool = False) -> "PlaneTensor":
        """K1 on device: (N, K) codes with ``nbits`` bits -> MSB-first planes."""
        _lib.require_cuda()
        c_d = _as_device_u8(codes)
        if c_d.dim() != 2:
            raise ValueError("codes must be a matrix")
        N, K = c_d.shape
        s_d = _as_device_f32(scales)
        ng = -(-K // group_size)
        if tuple(s_d.shape) != (N, ng):
            raise ValueError("scales shape %s != (%d, %d)" % (tuple(s_d.shape), N, ng))
        nplane_bytes = _lib.lib().mq_planes_bytes(N, K, nbits)
        planes = torch.empty(nplane_bytes // 4, dtype=torch.int32, device="cuda")
        ts = torch.empty(_lib.lib().mq_tscales_bytes(N, K, group_size) // 4, dtype=torch.float32,
                         device="cuda")
        sp = _lib.stream_ptr()
        _lib.call("mq_pack_planes", _lib.ptr(c_d), K, N, K, nbits, _lib.ptr(planes), sp)
        _lib.call("mq_tile_scales", _lib.ptr(s_d), N, K, group_size, _lib.ptr(ts), sp)
        return cls(planes, ts, N, K, group_size, nbits, is_child, scales_are_effective)

    @classmethod
    def random_parent(cls, N: int, K: int, group_size: int = 128, seed: int = 0,
                      scale_range=(0.005, 0.02)) -> "PlaneTensor":
        """Synthetic int8 parent generated on device (bench / model proxies)."""
        _lib.require_cuda()
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)
        codes = torch.randint(0, 256, (N, K), generator=g, device="cuda", dtype=torch.int32)
        codes = codes.to(torch.uint8)
        ng = -(-K // group_size)
        lo, hi = scale_range
        scales = torch.rand((N, ng), generator=g, device="cuda", dtype=torch.float32) * (hi - lo) + lo
        out = cls.from_codes(codes, 8, scales, group_size)
        del codes
        return out

    # -- geometry ----------------------------------------------------------
    @property
    def shape(self) -> tuple[int, int]:
        return (self.N, self.K)

    @property
    def nbytes(self) -> int:
        return self.planes.numel() * 4 + self.tscales.numel() * 4

    def _mode(self, r: int) -> tuple[int, float]:
        """(flags, out_scale) to read slice r from these planes."""
        if r not in LADDER:
            raise ValueError("unsupported bits")
        if self.is_child:
            if r != self.nbits:
                raise ValueError("a %d-bit child cannot serve %d bits" % (self.nbits, r))
            return _lib.MQ_CHILD, 1.0
        if r > self.nbits:
            raise ValueError("cannot slice %d bits out of %d" % (r, self.nbits))
        flags = _lib.MQ_CHILD if r == self.nbits else 0
        scale = 1.0 if self.scales_are_effective else float(1 << (self.nbits - r))
        return flags, scale

    def planes_read(self, r: int) -> int:
        """Planes a slice-r GEMV streams (r+1 in mode P, r in mode C / identity)."""
        flags, _ = self._mode(r)
        return r if flags & _lib.MQ_CHILD else r + 1

    # -- K2: slice / decode ------------------------------------------------
    def slice_codes(self, r: int) -> torch.Tensor:
        flags, _ = self._mode(r)
        out = torch.empty((self.N, self.K), dtype=torch.uint8, device="cuda")
        _lib.call("mq_slice", _lib.ptr(self.planes), self.N, self.K, r, int(bool(flags & _lib.MQ_CHILD)),
                  _lib.ptr(out), self.K, _lib.stream_ptr())
        return out

    def decode(self, r: int, values: bool = False) -> torch.Tensor:
        """fp32 dequantised weights (or int8 s - z) through the GEMV register path."""
        flags, scale = self._mode(r)
        child = int(bool(flags & _lib.MQ_CHILD))
        sp = _lib.stream_ptr()
        if values:
            out = torch.empty((self.N, self.K), dtype=torch.int8, device="cuda")
            _lib.call("mq_dequant", _lib.ptr(self.planes), None, self.N, self.K, self.G, r, child,
                      scale, _lib.ptr(out), None, self.K, sp)
        else:
            out = torch.empty((self.N, self.K), dtype=torch.float32, device="cuda")
            _lib.call("mq_dequant", _lib.ptr(self.planes), _lib.ptr(self.tscales), self.N, self.K,
                      self.G, r, child, scale, None, _lib.ptr(out), self.K, sp)
        return out

    def materialize_child(self, r: int) -> "PlaneTensor":
        """Mode C: an r-plane child sliced once from this parent (K2c)."""
        flags, scale = self._mode(r)
        if flags & _lib.MQ_CHILD:
            return self
        child = torch.empty(_lib.lib().mq_planes_bytes(self.N, self.K, r) // 4, dtype=torch.int32,
                            device="cuda")
        _lib.call("mq_materialize_child", _lib.ptr(self.planes), self.N, self.K, r, _lib.ptr(child),
                  _lib.stream_ptr())
        ts = self.tscales if scale == 1.0 else self.tscales * scale  # exact: power of two
        return PlaneTensor(child, ts, self.N, self.K, self.G, r, True, True)

    # -- K3 ----------------------------------------------------------------
    def gemv(self, X: torch.Tensor, r: int, out: torch.Tensor | None = None,
             out_dtype: torch.dtype | None = None, pdl: bool = False, stream=None) -> torch.Tensor:
        """Y = X @ dequant(slice_r).T for 1 <= B <= 32 rows (16 for fp32 X)."""
        flags, scale = self._mode(r)
        if X.dim() != 2 or X.shape[1] != self.K:
            raise ValueError("activations must be (batch, %d)" % self.K)
        if not X.is_cuda:
            raise ValueError("activations must be a CUDA tensor")
        if X.stride(1) != 1:
            X = X.contiguous()
        B = X.shape[0]
        if X.dtype == torch.float32:
            flags |= _lib.MQ_X_F32
        elif X.dtype != torch.bfloat16:
            raise ValueError("activations must be bfloat16 or float32")
        if out is None:
            od = out_dtype or (torch.float32 if X.dtype == torch.float32 else torch.bfloat16)
            out = torch.empty((B, self.N), dtype=od, device=X.device)
        if out.dtype == torch.float32:
            flags |= _lib.MQ_Y_F32
        elif out.dtype != torch.bfloat16:
            raise ValueError("output must be bfloat16 or float32")
        if out.stride(1) != 1 or out.shape != (B, self.N):
            raise ValueError("bad output tensor")
        if pdl:
            flags |= _lib.MQ_PDL
        sp = _lib.stream_ptr(stream)
        need = _lib.lib().mq_gemv_workspace_bytes(self.N, self.K, B, flags)
        ws = WORKSPACES.get(need, sp)
        _lib.call("mq_gemv", _lib.ptr(self.planes), _lib.ptr(self.tscales), _lib.ptr(X), X.stride(0),
                  _lib.ptr(out), out.stride(0), B, self.N, self.K, self.G, r, scale, flags,
                  _lib.ptr(ws), 0 if ws is None else ws.numel(), sp)
        return out

    def workspace_bytes(self, B: int, x_f32: bool = False) -> int:
        return _lib.lib().mq_gemv_workspace_bytes(self.N, self.K, B, _lib.MQ_X_F32 if x_f32 else 0)


def algorithmic_bytes(N: int, K: int, B: int, r: int, planes_read: int, G: int = 128,
                      x_bytes: int = 2, y_bytes: int = 2) -> int:
    """Bytes a GEMV must move: planes + fp32 scales + X + Y."""
    return N * K * planes_read // 8 + 4 * N * (-(-K // G)) + x_bytes * B * K + y_bytes * B * N
