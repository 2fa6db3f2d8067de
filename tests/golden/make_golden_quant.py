"""Golden vectors for the MatGPTQ quantiser row, made by
importing the reference itself.

Run in the build container (the only place /root/reference exists):

    NESTQUANT_NO_EXT=1 python tests/golden/make_golden_quant.py

Imports the unmodified reference package read-only from /root/reference/pkg/src
and writes tests/golden/quant_cases.npz:

* ``sel_*``: select_codes (gptq.py:119-140) over seeded matrices, every master
  width 2..8, ragged groups, exact grid points (ties), zeros, large values;
* ``fit_*``: fit_grid (grid.py:160-212): ragged final groups, zero groups,
  steps 1 / 5 / 51, several shrink_min;
* ``gq_*``: quantize_layer (gptq.py:143-226) with build_hessian /
  factor_inverse (gptq.py:67-94): codes, compensated snapshot and the
  diagnostics, several block sizes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    os.environ.setdefault("NESTQUANT_NO_EXT", "1")
    sys.path.insert(0, REF_SRC)
    from nestquant.gptq import build_hessian, factor_inverse, quantize_layer, select_codes
    from nestquant.grid import BitWidthSet, fit_grid

    out = {}
    rng = np.random.default_rng(20260217)

    def put_bits(prefix, bits):
        out[prefix + "_targets"] = np.asarray(bits.targets, dtype=np.int64)
        out[prefix + "_weights"] = np.asarray(bits.weights, dtype=np.float64)

    # ---- select_codes ---------------------------------------------------------
    sel_bits = [((2, 3, 4, 6, 8), (0.3, 0.7, 1.0, 1.5, 2.0)), ((8,), (1.0,)), ((2, 8), (1.0, 1.0)),
                ((4,), (1.0,)), ((2, 3), (10.0, 1.0)), ((3, 6), (0.25, 1.0)), ((2, 4, 5, 7), (1.0, 2.0, 0.5, 1.0)),
                ((2,), (1.0,)), ((2, 3, 4, 6, 8), (1.0, 1.0, 1.0, 1.0, 1.0))]
    for i, (t, w) in enumerate(sel_bits):
        bits = BitWidthSet(t, w)
        d_row, d_col, G = [(16, 300, 128), (7, 33, 32), (9, 64, 16), (5, 40, 8), (4, 6, 3),
                           (12, 130, 64), (6, 257, 128), (3, 20, 4), (20, 256, 128)][i]
        W = rng.standard_normal((d_row, d_col)) * rng.uniform(0.01, 3.0)
        ng = -(-d_col // G)
        scales = (np.abs(rng.standard_normal((d_row, ng))) * 0.05 + 1e-3).astype(np.float32)
        if i == 0:
            # exact grid points and midpoints (ties), zeros, saturating values
            cs = np.repeat(scales.astype(np.float64), G, axis=1)[:, :d_col]
            z = 1 << (bits.master - 1)
            W[0] = cs[0] * (np.arange(d_col) % (1 << bits.master) - z)
            W[1] = cs[1] * (np.arange(d_col) % (1 << bits.master) - z + 0.5)
            W[2] = 0.0
            W[3] = 1e3 * np.sign(rng.standard_normal(d_col))
        from nestquant.grid import QuantGrid

        grid = QuantGrid(master_bits=bits.master, group_size=G, scales=scales)
        out["sel%d_W" % i] = W
        out["sel%d_scales" % i] = scales
        out["sel%d_G" % i] = np.int64(G)
        put_bits("sel%d" % i, bits)
        out["sel%d_codes" % i] = np.asarray(select_codes(W, grid, bits), dtype=np.int64)
    out["sel_n"] = np.int64(len(sel_bits))

    # ---- fit_grid -------------------------------------------------------------
    fit_cases = [((2, 3, 4, 6, 8), (0.3, 0.7, 1.0, 1.5, 2.0), (8, 300), 128, 0.5, 51),
                 ((4,), (1.0,), (3, 33), 32, 0.5, 3),
                 ((2, 4), (1.0, 1.0), (1, 64), 64, 0.5, 51),
                 ((2, 3, 8), (1.0, 0.5, 2.0), (6, 96), 32, 0.5, 17),
                 ((2, 3, 8), (1.0, 0.5, 2.0), (6, 96), 32, 0.5, 1),
                 ((3, 4), (1.0, 1.0), (12, 24), 8, 0.3, 5),
                 ((8,), (1.0,), (5, 200), 128, 0.8, 11),
                 ((2, 3, 4, 6, 8), (1.0, 1.0, 1.0, 1.0, 1.0), (4, 1000), 256, 0.5, 21)]
    for i, (t, w, shape, G, smin, steps) in enumerate(fit_cases):
        bits = BitWidthSet(t, w)
        W = rng.standard_normal(shape) * rng.uniform(0.01, 2.0)
        if i == 0:
            W[1, :128] = 0.0  # a zero group: the scale floors
            W[2, 5] = 40.0    # one outlier per group
        out["fit%d_W" % i] = W
        out["fit%d_G" % i] = np.int64(G)
        out["fit%d_shrink" % i] = np.float64(smin)
        out["fit%d_steps" % i] = np.int64(steps)
        put_bits("fit%d" % i, bits)
        out["fit%d_scales" % i] = fit_grid(W, bits, G, shrink_min=smin, steps=steps).scales
    out["fit_n"] = np.int64(len(fit_cases))

    # ---- quantize_layer -------------------------------------------------------
    gq_cases = [((2, 3, 4, 6, 8), (0.3, 0.7, 1.0, 1.5, 2.0), 24, 260, 128, 128),
                ((3, 4, 8), (1.0, 1.0, 1.0), 24, 32, 32, 16),
                ((2, 4, 6), (1.0, 0.5, 1.5), 16, 48, 16, 16),
                ((4,), (1.0,), 48, 64, 32, 16),
                ((2, 8), (1.0, 1.0), 10, 200, 64, 40)]
    for i, (t, w, d_row, d_col, G, bs) in enumerate(gq_cases):
        bits = BitWidthSet(t, w)
        W = rng.standard_normal((d_row, d_col))
        X = rng.standard_normal((d_col, 2 * d_col))
        grid = fit_grid(W, bits, G, steps=9)
        H = build_hessian(X, 0.01)
        factor = factor_inverse(H, 0.01)
        layer, diag = quantize_layer(W, factor, grid, bits, block_size=bs, X=X)
        out["gq%d_W" % i] = W
        out["gq%d_X" % i] = X
        out["gq%d_G" % i] = np.int64(G)
        out["gq%d_bs" % i] = np.int64(bs)
        put_bits("gq%d" % i, bits)
        out["gq%d_scales" % i] = grid.scales
        out["gq%d_chol" % i] = factor.chol_upper
        out["gq%d_codes" % i] = layer.codes.astype(np.uint8)
        out["gq%d_comp" % i] = diag["compensated"]
        out["gq%d_recon" % i] = np.asarray([diag["recon"][r] for r in bits.targets])
        out["gq%d_obj" % i] = np.float64(diag["objective"])
    out["gq_n"] = np.int64(len(gq_cases))

    np.savez_compressed(os.path.join(HERE, "quant_cases.npz"), **out)
    print("wrote", os.path.join(HERE, "quant_cases.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
