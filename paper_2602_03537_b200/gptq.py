"""MatGPTQ quantiser on the GPU (drop-in for nestquant.gptq).

The same classes, functions, arguments and error texts as
/root/reference/pkg/src/nestquant/gptq.py; the work runs on the device:

* ``select_codes`` (gptq.py:104-140, the paper's Alg. 2): every weight
  scores all 2^c master codes against every target bit-width at once --
  ``mq_select_codes``, one warp per weight, float64, bit-identical;
* ``quantize_layer`` (gptq.py:143-226, Alg. 1): the blocked column loop.
  Inside a column block rows are independent, so ``mq_gptq_block`` runs the
  block's columns one warp per row (selection, averaged residual, rank-1
  updates) bit-identically; the update of the columns after the block,
  ``Wc[:, hi:] -= Err @ chol[lo:hi, hi:]``, is a plain float64 GEMM (cuBLAS
  through torch).  Its summation order differs from the host BLAS, so codes
  after the first block may differ from the reference's on near-ties
  (tests/test_gpu_quant.py bounds this);
* ``build_hessian`` / ``factor_inverse`` (gptq.py:67-94): float64 GEMM and
  Cholesky factorisations (cuBLAS / cuSOLVER through torch).

Inputs and outputs are numpy arrays, as in the reference; torch tensors are
accepted too.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import BitWidthSet, QuantGrid, _targets_args
from .slicing import NestedLayer

__all__ = ["QuantizeError", "CalibBatch", "HessianFactor", "build_hessian", "factor_inverse",
           "select_codes", "quantize_layer"]


class QuantizeError(RuntimeError):
    pass


def _dev64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


@dataclass
class CalibBatch:
    """Layer inputs, feature-major: X is (d_col, n_samples) (gptq.py:29-44)."""

    X: np.ndarray

    def __post_init__(self):
        self.X = np.ascontiguousarray(self.X, dtype=np.float64)
        if self.X.ndim != 2 or self.X.shape[1] < 1:
            raise QuantizeError("calibration batch must be (d_col, n>=1)")
        if not np.isfinite(self.X).all():
            raise QuantizeError("non-finite calibration data")

    @property
    def n_samples(self) -> int:
        return self.X.shape[1]


@dataclass
class HessianFactor:
    """Upper Cholesky factor of the inverse Hessian (gptq.py:47-64)."""

    chol_upper: np.ndarray
    damp_rel: float = 0.01
    damp_abs: float = 0.0

    def __post_init__(self):
        if (np.diag(np.asarray(self.chol_upper)) <= 0).any():
            raise QuantizeError("factorization failed: non-positive diagonal")

    @property
    def dim(self) -> int:
        return self.chol_upper.shape[0]


def build_hessian(X, damp_rel: float = 0.01) -> np.ndarray:
    """H = 2 X X^T + damp_rel * mean(diag(2 X X^T)) * I (gptq.py:67-79), on the GPU."""
    if damp_rel <= 0:
        raise QuantizeError("dampening must be positive")
    if isinstance(X, CalibBatch):
        X = X.X
    Xd = _dev64(X)
    G = 2.0 * (Xd @ Xd.T)
    mean_diag = float(torch.diagonal(G).mean())
    if mean_diag == 0.0:
        raise QuantizeError("degenerate calibration")
    G.diagonal().add_(damp_rel * mean_diag)
    return G.cpu().numpy()


def factor_inverse(H, damp_rel: float = 0.01) -> HessianFactor:
    """Upper Cholesky factor of H^-1 (gptq.py:82-94), on the GPU."""
    Hd = _dev64(H)
    L, info = torch.linalg.cholesky_ex(Hd)
    if int(info) != 0:
        raise QuantizeError("factorization failed")
    Hinv = torch.cholesky_inverse(L)
    Lu, info = torch.linalg.cholesky_ex(Hinv, upper=True)
    if int(info) != 0 or not bool(torch.isfinite(Lu).all()):
        raise QuantizeError("factorization failed")
    damp_abs = damp_rel * float(torch.diagonal(Hd).mean()) / (1.0 + damp_rel)
    return HessianFactor(chol_upper=Lu.cpu().numpy(), damp_rel=damp_rel, damp_abs=damp_abs)


def _select_device(Wd: torch.Tensor, grid: QuantGrid, bits: BitWidthSet) -> torch.Tensor:
    d_row, d_col = Wd.shape
    sc = torch.from_numpy(grid.scales).cuda()
    codes = torch.empty(d_row, d_col, dtype=torch.uint8, device="cuda")
    t, w, T = _targets_args(bits)
    _lib.call("mq_select_codes", _lib.ptr(Wd), Wd.stride(0), d_row, d_col, _lib.ptr(sc), sc.shape[1],
              grid.group_size, t, w, T, _lib.ptr(codes), codes.stride(0), _lib.stream_ptr(None))
    return codes


def select_codes(W, grid: QuantGrid, bits: BitWidthSet) -> np.ndarray:
    """Per weight, the master code minimising the weighted multi-bit error
    (gptq.py:119-140); ties go to the smallest code.  int64, like the reference."""
    Wd = _dev64(W)
    if Wd.dim() != 2:
        raise QuantizeError("weights must be a matrix")
    if not bool(torch.isfinite(Wd).all()):
        raise QuantizeError("non-finite weight")
    return _select_device(Wd, grid, bits).to(torch.int64).cpu().numpy()


def _master_values(c: int, r: int) -> torch.Tensor:
    """(S(q, r) - z) for every master code q, float64 on the device (grid.py:150-157)."""
    from .slicing import slice_code

    q = torch.arange(1 << c, device="cuda", dtype=torch.int64).to(torch.uint8)
    return torch.as_tensor(slice_code(q, c, r), device="cuda").to(torch.float64) - float(1 << (c - 1))


def quantize_layer(W, factor: HessianFactor, grid: QuantGrid, bits: BitWidthSet, block_size: int = 128,
                   name: str = "layer", X=None) -> tuple[NestedLayer, dict]:
    """Blocked column-serial quantisation with averaged cross-bit feedback
    (gptq.py:143-200).  Returns the nested layer plus diagnostics: the
    compensated weight snapshot and, when calibration inputs X (d_col, n) are
    given, per-bit-width reconstruction errors and their weighted sum."""
    W0 = _dev64(W)
    d_row, d_col = W0.shape
    if factor.dim != d_col:
        raise QuantizeError("factor dimension does not match layer")
    if block_size < 1:
        raise QuantizeError("block size must be >= 1")
    chol = _dev64(factor.chol_upper)
    sc = torch.from_numpy(grid.scales).cuda()
    Wc = W0.clone()
    codes = torch.empty(d_row, d_col, dtype=torch.uint8, device="cuda")
    comp = torch.empty_like(Wc)
    err = torch.empty(d_row, min(block_size, d_col), dtype=torch.float64, device="cuda")
    bad = torch.zeros((), dtype=torch.bool, device="cuda")
    t, w, T = _targets_args(bits)
    stream = _lib.stream_ptr(None)
    for lo in range(0, d_col, block_size):
        hi = min(lo + block_size, d_col)
        E = err[:, :hi - lo]
        _lib.call("mq_gptq_block", _lib.ptr(Wc), Wc.stride(0), d_row, d_col, lo, hi, _lib.ptr(sc), sc.shape[1],
                  grid.group_size, _lib.ptr(chol), chol.stride(0), t, w, T, _lib.ptr(codes), codes.stride(0),
                  _lib.ptr(comp), comp.stride(0), _lib.ptr(E), err.stride(0), stream)
        if hi < d_col:
            rest = Wc[:, hi:]
            rest.sub_(E @ chol[lo:hi, hi:])
            bad |= ~torch.isfinite(rest).all()
        bad |= ~torch.isfinite(E).all()
    if bool(bad):
        raise QuantizeError("numerical blowup")

    layer = NestedLayer(name=name, codes=codes.cpu().numpy(), grid=grid, bits=bits)
    diag: dict = {"compensated": comp.cpu().numpy()}
    if X is not None:
        Xd = _dev64(X)
        ref = W0 @ Xd
        cols = sc.to(torch.float64)[:, torch.arange(d_col, device="cuda") // grid.group_size]
        ci = codes.to(torch.int64)
        recon = {}
        for r in bits.targets:
            dq = cols * _master_values(bits.master, r)[ci]
            recon[r] = float(((dq @ Xd - ref) ** 2).sum())
        diag["recon"] = recon
        diag["objective"] = float(sum(lam * recon[r] for r, lam in zip(bits.targets, bits.weights)))
    return layer, diag
