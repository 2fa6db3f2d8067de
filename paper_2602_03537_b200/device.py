"""Device-resident bit-plane weights (the step-interleaved blob) and the GEMV.

A ``PlaneTensor`` owns one (N, K) layer in HBM: per (16-row tile, 256-column
step) a block of [group scales][MSB-first bit-plane slabs].  A
parent (``nplanes = c``, normally the int8 parent with c = 8) serves every
slice r <= c without repacking: slice r reads the scales and planes 0..r of
each block (mode P).  A child (``nplanes = r``) holds an already-sliced r-bit
code (mode C) and streams exactly r/8 of the parent's plane bytes.

Everything here is a thin shell over libmatq (include/matq.h); there is no
CPU compute path.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib

LADDER = (2, 3, 4, 6, 8)
MAX_GEMV_ROWS = 32
# linear(): K3 serves bf16 batches up to GEMV_DISPATCH_ROWS (measured crossover,
# profiles/r1_bench_batches.txt: at B = 32 K4 beats K3's NT = 4 tile), K4 (tcgen05)
# serves larger bf16 batches; gemv() itself accepts up to MAX_GEMV_ROWS.
GEMV_DISPATCH_ROWS = 16


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
_WS_NEED: dict[tuple[int, int, int, int], int] = {}


def _tuning_env() -> tuple:
    e = os.environ
    return (e.get("MQ_GEMV_SPLIT"), e.get("MQ_GEMV_WARPS"), e.get("MQ_GEMV_STAGES"),
            e.get("MQ_GEMV_STREAM"), e.get("MQ_GEMV_PAIR"))


def gemv_workspace_bytes(N: int, K: int, B: int, flags: int) -> int:
    """Cached mq_gemv_workspace_bytes (the launch path calls it every GEMV)."""
    # the C side honours tuning overrides (MQ_GEMV_*) that change the split
    key = (N, K, B, flags & _lib.MQ_X_F32, _tuning_env())
    v = _WS_NEED.get(key)
    if v is None:
        v = _WS_NEED[key] = _lib.lib().mq_gemv_workspace_bytes(N, K, B, flags)
    return v


_GEMM_WS: dict[tuple[int, int, int], int] = {}


def gemm_workspace_bytes(N: int, K: int, B: int) -> int:
    """Cached mq_gemm_workspace_bytes (split-K partials for small tile counts)."""
    key = (N, K, B)
    v = _GEMM_WS.get(key)
    if v is None:
        v = _GEMM_WS[key] = _lib.lib().mq_gemm_workspace_bytes(N, K, B, 0)
    return v


def reserve_workspace(nbytes: int, stream=None) -> None:
    WORKSPACES.get(int(nbytes), _lib.stream_ptr(stream))


class PlaneTensor:
    """Bit-plane blob (+ tiled scales when G != 128) of one layer on the GPU.

    ``nplanes`` is the number of stored planes: the master bit-width c of a
    parent (8 for the int8 parent), or r for an r-bit child.  ``master_bits``
    is the grid the scales live on; ``out_scale(r)`` = 2^(master_bits - r)
    unless the stored scales are already effective (a reference-style child).
    """

    def __init__(self, blob: torch.Tensor, tscales: torch.Tensor | None, N: int, K: int, G: int,
                 nplanes: int, master_bits: int, scales_are_effective: bool):
        self.blob = blob
        self.tscales = tscales
        self.N, self.K, self.G = int(N), int(K), int(G)
        self.nplanes = int(nplanes)
        self.master_bits = int(master_bits)
        self.scales_are_effective = bool(scales_are_effective)

    # -- construction ------------------------------------------------------
    @classmethod
    def from_codes(cls, codes, nbits: int, scales, group_size: int,
                   scales_are_effective: bool = False) -> "PlaneTensor":
        """K1 on device: (N, K) codes with ``nbits`` bits + (N, ng) scales -> blob."""
        _lib.require_cuda()
        if group_size < 32 or group_size % 32:
            raise ValueError("group size must be a multiple of 32")
        c_d = _as_device_u8(codes)
        if c_d.dim() != 2:
            raise ValueError("codes must be a matrix")
        N, K = c_d.shape
        s_d = _as_device_f32(scales)
        ng = -(-K // group_size)
        if tuple(s_d.shape) != (N, ng):
            raise ValueError("scales shape %s != (%d, %d)" % (tuple(s_d.shape), N, ng))
        L = _lib.lib()
        blob = torch.empty(L.mq_blob_bytes(N, K, group_size, nbits) // 4, dtype=torch.int32, device="cuda")
        ts = None
        if group_size != 128:
            ts = torch.empty(L.mq_tscales_bytes(N, K, group_size) // 4, dtype=torch.float32, device="cuda")
        _lib.call("mq_pack_blob", _lib.ptr(c_d), K, N, K, nbits, _lib.ptr(s_d), group_size,
                  _lib.ptr(blob), _lib.ptr(ts), _lib.stream_ptr())
        return cls(blob, ts, N, K, group_size, nbits, nbits, scales_are_effective)

    @staticmethod
    def random_parent_codes(N: int, K: int, group_size: int = 128, seed: int = 0,
                            scale_range=(0.005, 0.02), signed_rows: bool = False
                            ) -> tuple[torch.Tensor, torch.Tensor]:
        """The (codes uint8 (N, K), scales fp32 (N, ng)) random_parent packs, on device.

        Codes are uniform over [0, 255] (the reference's random_task,
        matmul.py:129-131).  Rounding slices of uniform codes are biased (mean
        s - z is -7.9 code units at r = 2, -1.9 at r = 3), which a chain of
        128 linears amplifies into an exponential blow-up of the activations'
        common mode; ``signed_rows`` gives every row's scales a random sign so
        that bias cancels across rows (the chained model proxies use it; the
        work per weight is unchanged)."""
        _lib.require_cuda()
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)
        codes = torch.randint(0, 256, (N, K), generator=g, device="cuda", dtype=torch.int32)
        codes = codes.to(torch.uint8)
        ng = -(-K // group_size)
        lo, hi = scale_range
        scales = torch.rand((N, ng), generator=g, device="cuda", dtype=torch.float32) * (hi - lo) + lo
        if signed_rows:
            sign = torch.randint(0, 2, (N, 1), generator=g, device="cuda", dtype=torch.int32) * 2 - 1
            scales = scales * sign.to(torch.float32)
        return codes, scales

    @classmethod
    def random_parent(cls, N: int, K: int, group_size: int = 128, seed: int = 0,
                      scale_range=(0.005, 0.02), signed_rows: bool = False) -> "PlaneTensor":
        """Synthetic int8 parent generated on device (bench / model proxies)."""
        codes, scales = cls.random_parent_codes(N, K, group_size, seed, scale_range, signed_rows)
        out = cls.from_codes(codes, 8, scales, group_size)
        del codes
        return out

    # -- geometry ----------------------------------------------------------
    @property
    def shape(self) -> tuple[int, int]:
        return (self.N, self.K)

    @property
    def nbytes(self) -> int:
        return self.blob.numel() * 4 + (0 if self.tscales is None else self.tscales.numel() * 4)

    def _check(self, r: int) -> float:
        """Validate slice r for this blob; returns the output scale."""
        if r not in LADDER:
            raise ValueError("unsupported bits")
        if r > self.nplanes:
            raise ValueError("cannot slice %d bits out of %d" % (r, self.nplanes))
        if r != self.nplanes and r + 1 > self.nplanes:
            raise ValueError("a %d-plane blob cannot serve %d bits" % (self.nplanes, r))
        return 1.0 if self.scales_are_effective else float(1 << (self.master_bits - r))

    def planes_read(self, r: int) -> int:
        """Planes a slice-r GEMV streams (r+1 in mode P, r in mode C / identity)."""
        self._check(r)
        return r if r == self.nplanes else r + 1

    # -- K2: slice / decode ------------------------------------------------
    def slice_codes(self, r: int) -> torch.Tensor:
        self._check(r)
        out = torch.empty((self.N, self.K), dtype=torch.uint8, device="cuda")
        _lib.call("mq_slice", _lib.ptr(self.blob), self.N, self.K, self.G, self.nplanes, r,
                  _lib.ptr(out), self.K, _lib.stream_ptr())
        return out

    def decode(self, r: int, values: bool = False) -> torch.Tensor:
        """fp32 dequantised weights (or int8 s - z) through the GEMV register path."""
        scale = self._check(r)
        sp = _lib.stream_ptr()
        if values:
            out = torch.empty((self.N, self.K), dtype=torch.int8, device="cuda")
            _lib.call("mq_dequant", _lib.ptr(self.blob), _lib.ptr(self.tscales), self.N, self.K,
                      self.G, self.nplanes, r, scale, _lib.ptr(out), None, self.K, sp)
        else:
            out = torch.empty((self.N, self.K), dtype=torch.float32, device="cuda")
            _lib.call("mq_dequant", _lib.ptr(self.blob), _lib.ptr(self.tscales), self.N, self.K,
                      self.G, self.nplanes, r, scale, None, _lib.ptr(out), self.K, sp)
        return out

    def materialize_child(self, r: int) -> "PlaneTensor":
        """Mode C: an r-plane child sliced once from this 8-plane parent (K2c)."""
        self._check(r)
        if r == self.nplanes:
            return self
        if self.nplanes != 8:
            raise ValueError("children are materialised from an 8-plane parent")
        child = torch.empty(_lib.lib().mq_blob_bytes(self.N, self.K, self.G, r) // 4,
                            dtype=torch.int32, device="cuda")
        _lib.call("mq_materialize_child", _lib.ptr(self.blob), self.N, self.K, self.G, r,
                  _lib.ptr(child), _lib.stream_ptr())
        return PlaneTensor(child, self.tscales, self.N, self.K, self.G, r, self.master_bits,
                           self.scales_are_effective)

    # -- K3 ----------------------------------------------------------------
    def gemv(self, X: torch.Tensor, r: int, out: torch.Tensor | None = None,
             out_dtype: torch.dtype | None = None, pdl: bool = False, stream=None) -> torch.Tensor:
        """Y = X @ dequant(slice_r).T for 1 <= B <= 32 rows (16 for fp32 X)."""
        scale = self._check(r)
        if X.dim() != 2 or X.shape[1] != self.K:
            raise ValueError("activations must be (batch, %d)" % self.K)
        if not X.is_cuda:
            raise ValueError("activations must be a CUDA tensor")
        if X.stride(1) != 1:
            X = X.contiguous()
        B = X.shape[0]
        flags = 0
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
        if out.stride(1) != 1 or tuple(out.shape) != (B, self.N):
            raise ValueError("bad output tensor")
        if pdl:
            flags |= _lib.MQ_PDL
        sp = _lib.stream_ptr(stream)
        need = gemv_workspace_bytes(self.N, self.K, B, flags)
        ws = WORKSPACES.get(need, sp)
        _lib.call("mq_gemv", _lib.ptr(self.blob), _lib.ptr(self.tscales), _lib.ptr(X), X.stride(0),
                  _lib.ptr(out), out.stride(0), B, self.N, self.K, self.G, self.nplanes, r, scale,
                  flags, _lib.ptr(ws), 0 if ws is None else ws.numel(), sp)
        return out

    # -- K4 ----------------------------------------------------------------
    def gemm(self, X: torch.Tensor, r: int, out: torch.Tensor | None = None,
             out_dtype: torch.dtype | None = None, pdl: bool = False, stream=None) -> torch.Tensor:
        """Y = X @ dequant(slice_r).T on the tcgen05 tensor cores (prefill, any B).

        X: bf16 (B, K), rows 16-byte aligned.  The dequantised weight is
        rounded to bf16 once (scale * (s - z)); accumulation is fp32.
        """
        scale = self._check(r)
        if self.G != 128:
            raise ValueError("the tensor-core path needs group size 128")
        if X.dim() != 2 or X.shape[1] != self.K:
            raise ValueError("activations must be (batch, %d)" % self.K)
        if not X.is_cuda or X.dtype != torch.bfloat16:
            raise ValueError("activations must be a bfloat16 CUDA tensor")
        if X.stride(1) != 1 or X.stride(0) % 8 or X.data_ptr() % 16:
            X = X.contiguous()
            if self.K % 8:
                raise ValueError("K must be a multiple of 8 for the tensor-core path")
        B = X.shape[0]
        if out is None:
            out = torch.empty((B, self.N), dtype=out_dtype or torch.bfloat16, device=X.device)
        flags = 0
        if out.dtype == torch.float32:
            flags |= _lib.MQ_Y_F32
        elif out.dtype != torch.bfloat16:
            raise ValueError("output must be bfloat16 or float32")
        if out.stride(1) != 1 or tuple(out.shape) != (B, self.N):
            raise ValueError("bad output tensor")
        if pdl:
            flags |= _lib.MQ_PDL
        sp = _lib.stream_ptr(stream)
        need = gemm_workspace_bytes(self.N, self.K, B)
        ws = WORKSPACES.get(need, sp)
        _lib.call("mq_gemm", _lib.ptr(self.blob), _lib.ptr(X), X.stride(0), _lib.ptr(out),
                  out.stride(0), B, self.N, self.K, self.G, self.nplanes, r, scale, flags,
                  _lib.ptr(ws), 0 if ws is None else ws.numel(), sp)
        return out

    def linear(self, X: torch.Tensor, r: int, out: torch.Tensor | None = None,
               out_dtype: torch.dtype | None = None, pdl: bool = False, stream=None) -> torch.Tensor:
        """Dispatch by batch: K3 (GEMV) up to GEMV_DISPATCH_ROWS rows, K4 (tcgen05 GEMM) above.

        fp32 activations or G != 128 stay on K3 (in 32/16-row chunks), which keeps
        the reference API's 1e-4 agreement (hi + lo bf16 split of fp32 X).
        """
        B = X.shape[0]
        if B <= GEMV_DISPATCH_ROWS or (X.dtype == torch.float32 and B <= 16):
            return self.gemv(X, r, out=out, out_dtype=out_dtype, pdl=pdl, stream=stream)
        if X.dtype == torch.bfloat16 and self.G == 128:
            return self.gemm(X, r, out=out, out_dtype=out_dtype, pdl=pdl, stream=stream)
        cap = 16 if X.dtype == torch.float32 else MAX_GEMV_ROWS
        if out is None:
            od = out_dtype or (torch.float32 if X.dtype == torch.float32 else torch.bfloat16)
            out = torch.empty((B, self.N), dtype=od, device=X.device)
        for lo in range(0, B, cap):
            self.gemv(X[lo:lo + cap], r, out=out[lo:lo + cap], pdl=pdl, stream=stream)
        return out

    def workspace_bytes(self, B: int, x_f32: bool = False) -> int:
        return _lib.lib().mq_gemv_workspace_bytes(self.N, self.K, B, _lib.MQ_X_F32 if x_f32 else 0)


def algorithmic_bytes(N: int, K: int, B: int, r: int, planes_read: int, G: int = 128,
                      x_bytes: int = 2, y_bytes: int = 2) -> int:
    """Bytes a GEMV must move: planes + fp32 scales + X + Y."""
    return N * K * planes_read // 8 + 4 * N * (-(-K // G)) + x_bytes * B * K + y_bytes * B * N


class StackProgram:
    """A whole decode step on the persistent K3S kernel (mq_stack_plan / mq_stack_run).

    ``layers``: (PlaneTensor, X, Y) in dependency order -- X of layer i+1 is
    (a column slice of) Y of layer i.  ``r``: one width for every layer, or a
    per-layer sequence (parents only; one kernel dispatching per layer).  X / Y
    bf16 CUDA tensors with unit column stride.  The host plan and the device
    layer table are built once; ``run()`` is one asynchronous,
    graph-capturable launch.
    """

    def __init__(self, layers, r, B: int, ops=None):
        """``ops``: optional per-layer activation prologue / output epilogue (None or a
        dict with xop, res_in, res_out, norm_w, eps, yop: mq_stack_layer's fused
        residual-add + RMSNorm / SiLU gating of the input, gated output)."""
        import ctypes

        _lib.require_cuda()
        L = _lib.lib()
        n = len(layers)
        arr = (_lib.StackLayer * n)()
        nplanes = None
        rs = [int(r)] * n if isinstance(r, int) else [int(x) for x in r]
        if len(rs) != n:
            raise ValueError("%d bit-widths for %d layers" % (len(rs), n))
        for i, (pt, X, Y) in enumerate(layers):
            scale = pt._check(rs[i])
            if pt.G != 128:
                raise ValueError("the stack kernel needs group size 128")
            if nplanes is None:
                nplanes = pt.nplanes
            elif pt.nplanes != nplanes:
                raise ValueError("mixed parent / child layers")
            if X.dtype != torch.bfloat16 or Y.dtype != torch.bfloat16 or X.stride(1) != 1 or Y.stride(1) != 1:
                raise ValueError("stack activations must be bf16 with unit column stride")
            arr[i] = _lib.StackLayer(_lib.ptr(pt.blob), X.data_ptr(), Y.data_ptr(), X.stride(0), Y.stride(0),
                                     pt.N, pt.K, scale, rs[i])
            op = ops[i] if ops else None
            if op:
                arr[i].xop = int(op.get("xop", 0))
                arr[i].yop = int(op.get("yop", 0))
                for key in ("res_in", "res_out"):
                    t = op.get(key)
                    if t is not None:
                        if t.dtype != torch.bfloat16 or t.stride(1) != 1:
                            raise ValueError("the residual must be bf16 with unit column stride")
                        setattr(arr[i], key, t.data_ptr())
                        arr[i].ldres = t.stride(0)
                if op.get("norm_w") is not None:
                    arr[i].norm_w = op["norm_w"].data_ptr()
                arr[i].eps = float(op.get("eps", 1e-5))
        r_plan = rs[0] if len(set(rs)) == 1 else 0
        if r_plan == 0 and nplanes != 8:
            raise ValueError("per-layer bit-widths need parent layers")
        self.plan = ctypes.create_string_buffer(L.mq_stack_plan_bytes())
        table = ctypes.create_string_buffer(L.mq_stack_table_bytes(n))
        ws = ctypes.c_size_t(0)
        _lib.call("mq_stack_plan", ctypes.cast(arr, ctypes.c_void_p), n, B, r_plan, nplanes, self.plan, table,
                  ctypes.byref(ws))
        self.table = torch.frombuffer(bytearray(table.raw), dtype=torch.uint8).cuda()
        self.ws = torch.zeros(max(ws.value, 1), dtype=torch.uint8, device="cuda")
        self._keep = (layers, ops)  # the tensors the table points at
        self.n_layers = n

    def run(self, stream=None) -> None:
        _lib.call("mq_stack_run", self.plan, _lib.ptr(self.table), _lib.ptr(self.ws), self.ws.numel(),
                  _lib.stream_ptr(stream))

    def launches(self, set_to: int | None = None) -> int:
        """The step counter behind the layer barriers (mq_stack_epoch): read it,
        or re-base it to ``set_to`` (synchronous)."""
        import ctypes

        v = ctypes.c_ulonglong(0 if set_to is None else int(set_to))
        _lib.call("mq_stack_epoch", self.plan, _lib.ptr(self.ws), self.ws.numel(), ctypes.byref(v),
                  0 if set_to is None else 1, _lib.stream_ptr())
        return int(v.value)
