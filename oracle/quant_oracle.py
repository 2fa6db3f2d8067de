"""CPU oracle for the MatGPTQ quantiser searches (TEST INFRASTRUCTURE ONLY).

Only tests/ and bench.py's CPU legs may import this module; the product
(paper_2602_03537_b200.gptq / grid.fit_grid) runs the CUDA kernels of
csrc/matq_quant.cu and never falls back here.

A numpy restatement of the reference's float64 searches, written candidate-
major (a running minimum over codes / alphas instead of the reference's
(rows, cols, codes) error cube), in the same per-element operation order so
the results are bit-identical:

* ``select_codes``   -- nestquant/gptq.py:104-140
* ``fit_grid``       -- nestquant/grid.py:160-212 (numpy's pairwise ``sum``
  over each group, as the reference's ``.sum(axis=2)``)
* ``quantize_layer`` -- nestquant/gptq.py:143-226 (blocked column loop; the
  trailing update is numpy's ``@``, i.e. the host BLAS, as in the reference)

Pinned by tests/test_oracle_quant.py against tests/golden/quant_cases.npz,
which tests/golden/make_golden_quant.py produced by importing the reference.
"""

from __future__ import annotations

import numpy as np

SCALE_FLOOR = 1e-12  # grid.py:20


def master_values(c: int, r: int) -> np.ndarray:
    """(slice_to_code(q, c, r) << (c - r)) - 2^(c-1) for q in [0, 2^c)
    (grid.py:150-157 with slicing.py:31-54's rounding rule)."""
    q = np.arange(1 << c, dtype=np.int64)
    k = c - r
    low = q if k == 0 else np.minimum((q + (1 << (k - 1))) >> k, (1 << r) - 1)
    return ((low << k) - (1 << (c - 1))).astype(np.float64)


def column_scales(scales: np.ndarray, G: int, d_col: int) -> np.ndarray:
    return np.asarray(scales, dtype=np.float32)[:, np.arange(d_col) // G].astype(np.float64)


def select_codes(W, scales, G, targets, weights) -> np.ndarray:
    """Per weight, the master code minimising sum_t lam_t (w - s mv_t[q])^2
    (first minimum)."""
    W = np.asarray(W, dtype=np.float64)
    c = int(targets[-1])
    s = column_scales(scales, G, W.shape[1])
    tabs = [(float(lam), master_values(c, int(r))) for r, lam in zip(targets, weights)]
    best = np.full(W.shape, np.inf)
    code = np.zeros(W.shape, dtype=np.int64)
    for q in range(1 << c):
        err = np.zeros(W.shape)
        for lam, mv in tabs:
            d = W - s * mv[q]
            err = err + lam * (d * d)
        take = err < best
        best = np.where(take, err, best)
        code = np.where(take, q, code)
    return code


def _round_half_away(x):
    return np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5))


def fit_grid(W, targets, weights, G, shrink_min=0.5, steps=51) -> np.ndarray:
    """float32 (d_row, n_groups) shrink-searched scales."""
    W = np.asarray(W, dtype=np.float64)
    c = int(targets[-1])
    z, qmax = 1 << (c - 1), (1 << c) - 1
    d_row, d_col = W.shape
    ng = -(-d_col // G)
    alphas = np.linspace(1.0, shrink_min, steps)
    tabs = [(float(lam), master_values(c, int(r))) for r, lam in zip(targets, weights)]
    out = np.empty((d_row, ng))
    for g in range(ng):
        Wg = np.ascontiguousarray(W[:, g * G:min((g + 1) * G, d_col)])
        base = np.maximum(np.abs(Wg).max(axis=1) / float(z - 1), SCALE_FLOOR)
        best = np.full(d_row, np.inf)
        pick = np.zeros(d_row)
        for i, a in enumerate(alphas):
            s = (a * base)[:, None]
            q = np.clip(_round_half_away(Wg / s + z), 0, qmax).astype(np.int64)
            obj = np.zeros(d_row)
            for lam, mv in tabs:
                d = Wg - s * mv[q]
                obj = obj + lam * np.ascontiguousarray(d * d).sum(axis=1)
            take = (obj < best) if i else np.ones(d_row, dtype=bool)
            best = np.where(take, obj, best)
            pick = np.where(take, s[:, 0], pick)
        out[:, g] = pick
    return np.maximum(out.astype(np.float32), np.float32(SCALE_FLOOR))


def quantize_layer(W, chol, scales, G, targets, weights, block_size=128):
    """(codes uint8, compensated float64) of the blocked column loop."""
    Wc = np.array(W, dtype=np.float64, copy=True)
    d_row, d_col = Wc.shape
    c = int(targets[-1])
    s_all = column_scales(scales, G, d_col)
    tabs = [(float(lam), master_values(c, int(r))) for r, lam in zip(targets, weights)]
    nt = float(len(tabs))
    codes = np.empty((d_row, d_col), dtype=np.uint8)
    comp = np.empty_like(Wc)
    with np.errstate(over="ignore", invalid="ignore"):
        for lo in range(0, d_col, block_size):
            hi = min(lo + block_size, d_col)
            E = np.zeros((d_row, hi - lo))
            for j in range(lo, hi):
                w = Wc[:, j].copy()
                comp[:, j] = w
                q = select_codes(w[:, None], s_all[:, j:j + 1].astype(np.float32), 1, targets, weights)[:, 0]
                codes[:, j] = q
                s = s_all[:, j]
                resid = np.zeros(d_row)
                for _, mv in tabs:
                    resid = resid + (w - s * mv[q])
                e = (resid / nt) / chol[j, j]
                E[:, j - lo] = e
                if j + 1 < hi:
                    Wc[:, j + 1:hi] -= e[:, None] * chol[j, j + 1:hi][None, :]
            if hi < d_col:
                Wc[:, hi:] -= E @ chol[lo:hi, hi:]
            if not np.isfinite(Wc[:, hi:]).all() or not np.isfinite(E).all():
                raise FloatingPointError("numerical blowup")
    return codes, comp
