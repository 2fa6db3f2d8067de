"""Quantiser searches on a Llama-3.1-8B-sized layer:
GPU time of select_codes / fit_grid / quantize_layer vs the numpy oracle
(the reference's algorithm) on a bounded row sample, scaled per weight."""
import json
import sys
import time

import numpy as np
import torch

import paper_2602_03537_b200 as mq
from paper_2602_03537_b200 import _lib
from paper_2602_03537_b200.grid import _targets_args


def dev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    N, K = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4096, 4096)
    rng = np.random.default_rng(0)
    bits = mq.BitWidthSet((2, 3, 4, 6, 8), (1.0, 1.0, 1.0, 1.0, 1.0))
    W = rng.standard_normal((N, K)) * 0.02
    Wd = torch.from_numpy(W).cuda()
    t, w, T = _targets_args(bits)
    alphas = torch.from_numpy(np.linspace(1.0, 0.5, 51)).cuda()
    ng = K // 128
    sc = torch.empty(N, ng, dtype=torch.float32, device="cuda")
    codes = torch.empty(N, K, dtype=torch.uint8, device="cuda")
    fit = lambda: _lib.call("mq_fit_grid", _lib.ptr(Wd), K, N, K, 128, t, w, T, _lib.ptr(alphas), 51,  # noqa: E731
                            _lib.ptr(sc), _lib.stream_ptr(None))
    sel = lambda: _lib.call("mq_select_codes", _lib.ptr(Wd), K, N, K, _lib.ptr(sc), ng, 128, t, w, T,  # noqa: E731
                            _lib.ptr(codes), K, _lib.stream_ptr(None))
    t_fit = dev_time(fit)
    t_sel = dev_time(sel)
    grid = mq.QuantGrid(8, 128, sc.cpu().numpy())
    X = rng.standard_normal((K, 256))
    factor = mq.factor_inverse(mq.build_hessian(X, 0.01), 0.01)
    mq.quantize_layer(W[:256], factor, mq.QuantGrid(8, 128, grid.scales[:256]), bits)  # warm (cuBLAS, modules)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mq.quantize_layer(W, factor, grid, bits, block_size=128)
    t_gq = time.perf_counter() - t0
    # CPU: the numpy oracle on a row sample
    from oracle import quant_oracle as Q

    rows = 64
    c0 = time.perf_counter()
    Q.select_codes(W[:rows], grid.scales[:rows], 128, bits.targets, bits.weights)
    c_sel = (time.perf_counter() - c0) * N / rows
    c0 = time.perf_counter()
    Q.fit_grid(W[:rows], bits.targets, bits.weights, 128)
    c_fit = (time.perf_counter() - c0) * N / rows
    c0 = time.perf_counter()
    Q.quantize_layer(W[:rows], factor.chol_upper, grid.scales[:rows], 128, bits.targets, bits.weights)
    c_gq = (time.perf_counter() - c0) * (N / rows)
    print(json.dumps({"layer": [N, K], "targets": list(bits.targets), "G": 128, "steps": 51,
                      "gpu_s": {"fit_grid": t_fit, "select_codes": t_sel, "quantize_layer": t_gq},
                      "cpu_oracle_s_est": {"fit_grid": c_fit, "select_codes": c_sel,
                                           "quantize_layer": c_gq,
                                           "sample": "%d of %d rows, full width, scaled by rows" % (rows, N)},
                      "weights_per_s": {"select_codes": N * K / t_sel, "fit_grid": N * K / t_fit}}))


if __name__ == "__main__":
    main()
