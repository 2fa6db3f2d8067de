"""Benchmark: Llama-3.1-8B decode tok/s per bit-width + sliced-GEMV roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--bits 4] [--batch 1]
    python bench.py --impl reference ...          # the reference's CPU path

One step = one decode token through every linear of the Llama-3.1-8B stack
(32 blocks x {qkv, o, gate_up, down}, 6.98 B int8-parent weights resident in
HBM, each sliced on the fly to r bits), replayed as one CUDA graph of K3
launches.  Synthetic random-init parents; the stack's weights (>= 2.6 GB per
step at r = 2) are far larger than the 126 MB L2, so every step is L2-cold.

Printed JSON (one line, rank 0):
  value       tok/s at the headline bit-width (--bits, default 4), device-resident
              activations, K steps timed with CUDA events (max over ranks)
  e2e         same metric through LinearStack.decode(): pinned host x -> H2D ->
              graph -> D2H of y, every step
  per_bits    tok/s for every r on the ladder (mode P; mode C children too)
  roofline    dominant kernel (gate_up GEMV, 28672 x 4096): algorithmic bytes per
              launch / CUDA-event duration vs MEASURED_PEAKS.json HBM GB/s
  cpu_baseline  the reference's own compiled kernel (oracle/_ref) on the host
              cores for a bounded sample (one block, extrapolated x32)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Llama-3.1-8B decode tok/s per bit-width; sliced-GEMV HBM GB/s vs roofline"
UNIT = "tok/s"
LADDER = (2, 3, 4, 6, 8)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling through NVML."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._active = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            if self._active.is_set():
                try:
                    self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                    self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    pass
            time.sleep(0.02)

    def active(self, on: bool):
        (self._active.set if on else self._active.clear)()

    def summary(self):
        self._stop.set()
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def _shapes():
    """paper_2602_03537_b200/shapes.py loaded by path: the reference arm shares
    the workload definition without importing the package (which maps libmatq.so)."""
    import importlib.util

    if "_mq_shapes" not in sys.modules:
        spec = importlib.util.spec_from_file_location(
            "_mq_shapes", os.path.join(ROOT, "paper_2602_03537_b200", "shapes.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules["_mq_shapes"] = mod
        spec.loader.exec_module(mod)
    return sys.modules["_mq_shapes"]


def workload_config(model: str, n_blocks: int, bits: int, batch: int, world: int) -> dict:
    """The config both arms report (same workload, same keys, same values)."""
    sh = _shapes()
    shape = sh.SHAPES[model]
    dims = ", ".join("%s %dx%d" % ((k,) + sh.full_layer_dims(shape, k)) for k in sh.KINDS)
    return {"workload": "%s linear stack decode: %d blocks x {%s}, int8 parent sliced to r bits "
                        "(rounding MSB slice), G=128" % (model, n_blocks, dims),
            "model": model, "bits": bits, "batch": batch, "group_size": 128,
            "parallelism": "tp%d" % world}


# ------------------------------------------------------------ CPU baseline --
class CpuReference:
    """One Llama-3.1-8B block (qkv, o, gate_up, down) on the host cores.

    r in {2,3,4}: the reference's compiled nq_gemv/nq_gemm (oracle/_ref, driven
    as kernels/_core.pyx:24-64 drives it); with threads > 1 the rows are spread
    over host threads (the kernel walks rows independently, packed_kernels.c:88;
    ctypes releases the GIL), threads = 1 is the reference as shipped (one
    core, _core.pyx:47-63).  r in {6,8}: the reference has no packed kernel
    (matmul.py:55-56); its bench baseline, a dense fp32 GEMV on the
    dequantised child (matmul.py:164-165), is used instead.
    Preparation (slice + pack) is untimed, as in the reference bench.
    ``step_seconds`` runs a whole decode step: the block's four linears once per
    model block (32 for Llama-3.1-8B; the blocks share shapes, so one block's
    weights are reused -- 110 MB at r = 4, beyond any host LLC).
    """

    def __init__(self, r: int, batch: int, threads: int, model: str = "Llama-3.1-8B"):
        import numpy as np
        from concurrent.futures import ThreadPoolExecutor

        from oracle import oracle as O

        sh = _shapes()
        shape = sh.SHAPES[model]
        self.r, self.threads, self.O = r, threads, O
        self.n_blocks = shape.n_layers
        rng = np.random.default_rng(0)
        self.layers = []
        for kind in sh.KINDS:
            N, K = sh.full_layer_dims(shape, kind)
            parent = rng.integers(0, 256, size=(N, K), dtype=np.uint8)
            scales = rng.uniform(0.005, 0.02, size=(N, K // 128)).astype(np.float32)
            child = O.slice_codes(parent, 8, r)
            seff = O.scale_eff(scales, 8, r)
            X = rng.standard_normal((batch, K)).astype(np.float32)
            if r <= 4:
                base, b2, b3 = O.pack_child(child, r)
                self.layers.append(("packed", N, base, b2, b3, seff, X))
            else:
                W = O.dense_f32(child, seff, 128, r)
                self.layers.append(("dense", N, W, None, None, None, X))
            del parent, child
        self.ref = O.RefKernels() if r <= 4 else None
        self.pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
        self.kind = "reference" if r <= 4 else "port"
        self.backend = (self.ref.backend_name() if self.ref
                        else "dense-fp32 GEMV (oracle C; the reference bench's baseline)")

    def _layer(self, ly):
        kind, N = ly[0], ly[1]
        if self.pool is None:
            if kind == "packed":
                _, _, base, b2, b3, seff, X = ly
                self.ref.packed_matmul(base, b2, b3, seff, X, self.r, 128)
            else:
                self.O.dense_gemm(ly[6], ly[2])
            return
        step = -(-N // max(1, self.threads * 4))
        bounds = [(lo, min(N, lo + step)) for lo in range(0, N, step)]
        if kind == "packed":
            _, _, base, b2, b3, seff, X = ly
            futs = [self.pool.submit(self.ref.packed_matmul, base, b2, b3, seff, X, self.r, 128,
                                     rows=b) for b in bounds]
        else:
            _, _, W, _, _, _, X = ly
            futs = [self.pool.submit(self.O.dense_gemm, X, W[lo:hi]) for lo, hi in bounds]
        for f in futs:
            f.result()

    def block_seconds(self) -> float:
        t0 = time.perf_counter()
        for ly in self.layers:
            self._layer(ly)
        return time.perf_counter() - t0

    def step_seconds(self) -> float:
        """One decode step: every block's four linears (no extrapolation)."""
        t0 = time.perf_counter()
        for _ in range(self.n_blocks):
            for ly in self.layers:
                self._layer(ly)
        return time.perf_counter() - t0

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def run_reference(args):
    """The reference arm: the reference's own CPU implementation of the path
    (oracle/_ref = its packed_kernels.c, compiled unmodified; r in {6, 8}: its
    bench's dense fp32 baseline), all host threads, on the GPU arm's workload,
    config, metric and unit.  Every timed step is a whole decode step (32
    blocks x 4 linears).  Nothing from paper_2602_03537_b200 is imported."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    r = args.bits
    ref = CpuReference(r, args.batch, threads, args.model)
    samples = []
    t_all = time.perf_counter()
    for i in range(args.warmup + args.steps):
        t = ref.step_seconds() if i >= args.warmup else ref.block_seconds()  # warm-up: one block
        if i >= args.warmup:
            samples.append(t)
    ref.close()
    total = sum(samples)
    tok_s = args.batch * len(samples) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / len(samples) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic",
        "config": workload_config(args.model, ref.n_blocks, r, args.batch, args.gpus),
        "cpu_baseline": {"value": tok_s, "unit": UNIT, "cores": threads, "kind": ref.kind,
                         "sample": "every timed step is one whole decode step: %d blocks x 4 linears, all "
                                   "rows (one block's weights reused per block); warm-up steps run one "
                                   "block; backend %s, rows split over %d threads" % (
                                       ref.n_blocks, ref.backend, threads)},
        "e2e": {"value": tok_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
    }
    print(json.dumps(line), flush=True)
    return 0


def c1_leg(torch, mq, clocks, peak, cpu: bool, bits=(8, 4, 2), N=4096, K=4096, reps=10):
    """BASELINE C1, the case the reference's own bench runs (matmul.py:123-192,
    cli.py:237-245): one 4096x4096 linear, int8 parent sliced to r, G = 128,
    B = 1.  L2-cold: 40 weight replicas (each launch reads >= 6.5 MiB; 40 x
    that >= 2 x the 126 MB L2) cycled inside one CUDA graph of K3 launches
    (PDL).  Beside it, the reference's compiled kernel on 1 core (r in {4, 2};
    r = 8: its bench's dense fp32 GEMV), median of 7 after 1 warm-up
    (matmul.py:138-145)."""
    import numpy as np

    from paper_2602_03537_b200.device import algorithmic_bytes

    nrep = 40
    pts = [mq.PlaneTensor.random_parent(N, K, 128, seed=1000 + i) for i in range(nrep)]
    X = torch.randn(1, K, device="cuda").to(torch.bfloat16)
    Y = torch.empty(1, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    out = {}
    for r in bits:
        with torch.cuda.stream(s):
            for pt in pts:
                pt.gemv(X, r, out=Y, pdl=True, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for pt in pts:
                pt.gemv(X, r, out=Y, pdl=True, stream=s)
        with torch.cuda.stream(s):
            for _ in range(3):
                g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks.active(True)
        e0.record(s)
        with torch.cuda.stream(s):
            for _ in range(reps):
                g.replay()
        e1.record(s)
        e1.synchronize()
        clocks.active(False)
        t = e0.elapsed_time(e1) / 1e3 / (reps * nrep)
        nb = algorithmic_bytes(N, K, 1, r, pts[0].planes_read(r), 128)
        rec = {"us": t * 1e6, "GBps": nb / t / 1e9, "frac": nb / t / 1e9 / peak, "bytes": nb,
               "ideal_r_bytes": algorithmic_bytes(N, K, 1, r, r, 128)}
        if cpu:
            from oracle import oracle as O

            rng = np.random.default_rng(0)
            parent = rng.integers(0, 256, size=(N, K), dtype=np.uint8)
            scales = rng.uniform(0.005, 0.02, size=(N, K // 128)).astype(np.float32)
            xs = rng.standard_normal((1, K)).astype(np.float32)
            child = O.slice_codes(parent, 8, r)
            seff = O.scale_eff(scales, 8, r)
            if r <= 4:
                ref = O.RefKernels()
                base, b2, b3 = O.pack_child(child, r)
                fn = lambda: ref.packed_matmul(base, b2, b3, seff, xs, r, 128)  # noqa: E731
                kind = "reference (%s)" % ref.backend_name()
            else:
                W = O.dense_f32(child, seff, 128, r)
                fn = lambda: O.dense_gemm(xs, W)  # noqa: E731
                kind = "port (dense fp32 GEMV, the reference bench baseline)"
            fn()
            ts = []
            for _ in range(7):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            rec["cpu_us"] = statistics.median(ts) * 1e6
            rec["cpu_kind"] = kind
            rec["cpu_cores"] = 1
            rec["vs_cpu"] = rec["cpu_us"] / rec["us"]
        out["r%d" % r] = rec
        del g
    del pts
    torch.cuda.empty_cache()
    return {"shape": [N, K], "batch": 1, "group_size": 128,
            "l2": "cold: 40 replicas cycled in one graph", "per_bits": out}


def sweep_leg(torch, stack, clocks, peak, batches, configs, steps=10, warmup=3):
    """Decode batch sweep of a LinearStack (BASELINE C2 uniform r / C3
    heterogeneous): the default dispatch (K3S or the per-layer K3 graph)."""
    out = {}
    for B in batches:
        stack.set_batch(B)
        for label, cfg in configs:
            stack.capture(cfg)
            for _ in range(warmup):
                stack.step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            clocks.active(True)
            e0.record(stack.stream)
            for _ in range(steps):
                stack.step()
            e1.record(stack.stream)
            e1.synchronize()
            clocks.active(False)
            t = e0.elapsed_time(e1) / 1e3 / steps
            nb = stack.step_bytes(stack.config)
            out["B%d_%s" % (B, label)] = {
                "tok_s": B / t, "ms_per_step": t * 1e3, "GBps": nb / t / 1e9, "frac": nb / t / 1e9 / peak,
                "path": "K3S" if stack.launches_per_step() == 1 else "K3 graph"}
    stack.set_batch(1)
    return out


def graph_seconds(torch, fns, reps, clocks=None):
    """Device seconds per call of ``fns`` (each fn(stream)): the calls are
    captured once into a CUDA graph (no host launch cost in the timed region),
    replayed ``reps`` times between CUDA events on the capture stream."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for fn in fns:
            fn(s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for fn in fns:
            fn(s)
    with torch.cuda.stream(s):
        for _ in range(2):
            g.replay()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.active(True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    e1.record(s)
    e1.synchronize()
    if clocks:
        clocks.active(False)
    del g
    return e0.elapsed_time(e1) / 1e3 / (reps * len(fns))


def prefill_leg(torch, mq, clocks, batches=(64, 256, 1024), bits=(4, 8), reps=10):
    """Qwen3-14B linears through K4 (tcgen05) at prefill batches: TFLOP/s per
    layer and for the 4-layer block, vs the measured bf16 peak and a dense
    bf16 cuBLAS GEMM of the same shape.  Both sides rotate 3 weight copies
    (L2-cold) inside one CUDA graph (device time, no host launch cost)."""
    from paper_2602_03537_b200.model import QWEN3_14B, KINDS, full_layer_dims

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        pk = json.load(f)
    tf_peak = float(pk.get("bf16_tflops", 1631.2))

    res = {}
    for kind in KINDS:
        N, K = full_layer_dims(QWEN3_14B, kind)
        pts = [mq.PlaneTensor.random_parent(N, K, seed=i) for i in range(3)]
        Wd = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
        for B in batches:
            X = torch.randn(B, K, device="cuda").to(torch.bfloat16)
            Y = torch.empty(B, N, device="cuda", dtype=torch.bfloat16)
            dense = graph_seconds(torch, [lambda s, w=w: torch.matmul(X, w.t(), out=Y) for w in Wd], reps, clocks)
            for r in bits:
                t = graph_seconds(torch, [lambda s, pt=pt: pt.gemm(X, r, out=Y, pdl=True, stream=s)
                                          for pt in pts], reps, clocks)
                res[(kind, B, r)] = (t, dense, 2.0 * B * N * K)
        del pts, Wd
        torch.cuda.empty_cache()
    out = {"model": "Qwen3-14B", "peak_tflops": tf_peak, "peak_kind": "measured bf16 (burst)",
           "timing": "CUDA graph of 3 rotated weight copies per side (L2-cold), device time",
           "per_layer": {}, "block": {}}
    for (kind, B, r), (t, dense, fl) in res.items():
        out["per_layer"]["%s_B%d_r%d" % (kind, B, r)] = {
            "us": t * 1e6, "tflops": fl / t / 1e12, "frac": fl / t / 1e12 / tf_peak,
            "dense_bf16_us": dense * 1e6, "vs_dense": dense / t}
    for B in batches:
        for r in bits:
            t = sum(res[(k, B, r)][0] for k in KINDS)
            d = sum(res[(k, B, r)][1] for k in KINDS)
            fl = sum(res[(k, B, r)][2] for k in KINDS)
            out["block"]["B%d_r%d" % (B, r)] = {
                "us": t * 1e6, "tflops": fl / t / 1e12, "frac": fl / t / 1e12 / tf_peak,
                "tok_s_40_blocks": B / (40 * t), "vs_dense": d / t}
    return out


# ------------------------------------------------------------------ GPU arm --
def quant_leg(torch, mq, cpu: bool, N=4096, K=4096, G=128, cpu_rows=16):
    """the MatGPTQ quantiser searches (csrc/matq_quant.cu) on
    a Llama-3.1-8B-sized layer, targets {2,3,4,6,8}: device time of
    select_codes / fit_grid (CUDA events, inputs resident) and of
    quantize_layer through the numpy drop-in API; the oracle (the reference's
    algorithm in numpy) on a row sample, scaled by rows."""
    import time

    import numpy as np

    from paper_2602_03537_b200 import _lib
    from paper_2602_03537_b200.grid import _targets_args

    rng = np.random.default_rng(0)
    bits = mq.BitWidthSet((2, 3, 4, 6, 8), (1.0, 1.0, 1.0, 1.0, 1.0))
    W = rng.standard_normal((N, K)) * 0.02
    Wd = torch.from_numpy(W).cuda()
    t, w, T = _targets_args(bits)
    alphas = torch.from_numpy(np.linspace(1.0, 0.5, 51)).cuda()
    ng = -(-K // G)
    sc = torch.empty(N, ng, dtype=torch.float32, device="cuda")
    codes = torch.empty(N, K, dtype=torch.uint8, device="cuda")

    def fit():
        _lib.call("mq_fit_grid", _lib.ptr(Wd), K, N, K, G, t, w, T, _lib.ptr(alphas), 51, _lib.ptr(sc),
                  _lib.stream_ptr(None))

    def sel():
        _lib.call("mq_select_codes", _lib.ptr(Wd), K, N, K, _lib.ptr(sc), ng, G, t, w, T, _lib.ptr(codes), K,
                  _lib.stream_ptr(None))

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

    t_fit, t_sel = dev_time(fit), dev_time(sel)
    grid = mq.QuantGrid(8, G, sc.cpu().numpy())
    X = rng.standard_normal((K, 256))
    factor = mq.factor_inverse(mq.build_hessian(X, 0.01), 0.01)
    mq.quantize_layer(W[:256], factor, mq.QuantGrid(8, G, grid.scales[:256]), bits)  # warm cuBLAS
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mq.quantize_layer(W, factor, grid, bits, block_size=128)
    t_gq = time.perf_counter() - t0
    out = {"layer": [N, K], "targets": list(bits.targets), "group_size": G, "fit_steps": 51,
           "device_s": {"select_codes": t_sel, "fit_grid": t_fit},
           "api_s": {"quantize_layer": t_gq,
                     "note": "numpy in/out: includes 2x134 MB H2D and 134 MB D2H of float64"},
           "weights_per_s": {"select_codes": N * K / t_sel, "fit_grid": N * K / t_fit},
           "parity": "select_codes / fit_grid bit-exact vs the reference (tests/test_gpu_quant.py)"}
    if cpu:
        from oracle import quant_oracle as Q

        c0 = time.perf_counter()
        Q.select_codes(W[:cpu_rows], grid.scales[:cpu_rows], G, bits.targets, bits.weights)
        c_sel = (time.perf_counter() - c0) * N / cpu_rows
        c0 = time.perf_counter()
        Q.fit_grid(W[:cpu_rows], bits.targets, bits.weights, G)
        c_fit = (time.perf_counter() - c0) * N / cpu_rows
        out["cpu_baseline_s"] = {"select_codes": c_sel, "fit_grid": c_fit, "kind": "port", "cores": 1,
                                 "sample": "%d of %d rows, scaled by rows (numpy oracle)" % (cpu_rows, N)}
    del Wd, codes, sc
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="matq", choices=["matq", "reference"])
    ap.add_argument("--bits", type=int, default=4, choices=LADDER)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=None, help="debug: fewer blocks")
    ap.add_argument("--no-sweep", action="store_true", help="headline r only (no per-bits, mode C)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-hetero", action="store_true", help="skip the C3 heterogeneous-config leg")
    ap.add_argument("--no-prefill", action="store_true", help="skip the C4 tcgen05 prefill leg")
    ap.add_argument("--no-full", action="store_true", help="skip the full-model decode leg")
    ap.add_argument("--no-quant", action="store_true", help="skip the quantiser-search leg")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 single-layer leg")
    ap.add_argument("--no-c2", action="store_true", help="skip the C2 / C3 batch sweeps")
    ap.add_argument("--model", default="Llama-3.1-8B", help="Llama-3.1-8B | Qwen3-14B | Phi-3-Medium")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torch.distributed.run
        import socket
        import subprocess

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
               str(args.gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
               os.path.abspath(__file__)] + sys.argv[1:]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")  # rank / channel / NVLS lines go to stderr
        return subprocess.call(cmd, env=env)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pg = dist.group.WORLD if world > 1 else None

    import paper_2602_03537_b200 as mq
    from paper_2602_03537_b200.device import algorithmic_bytes
    from paper_2602_03537_b200.model import SHAPES, LinearStack

    peak, peak_kind = _peaks()
    shape = SHAPES[args.model]
    stack = LinearStack(shape, batch=args.batch, tp=world, rank=rank, process_group=pg,
                        n_layers=args.layers)
    n_blocks = stack.n_layers
    clocks = ClockSampler(local)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def time_steps(fn, k):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks.active(True)
        e0.record(stack.stream)
        for _ in range(k):
            fn()
        e1.record(stack.stream)
        barrier()
        clocks.active(False)
        return max_over_ranks(e0.elapsed_time(e1) / 1e3)

    results = {}
    order = [args.bits] + ([r for r in LADDER if r != args.bits] if not args.no_sweep else [])
    head_launches = None
    for r in order:
        stack.capture(r)
        if head_launches is None:
            head_launches = stack.launches_per_step()
        for _ in range(args.warmup):
            stack.step()
        secs = time_steps(stack.step, args.steps)
        results[r] = {"tok_s": args.batch * args.steps / secs, "ms_per_step": secs / args.steps * 1e3,
                      "bytes_per_step": stack.step_bytes(stack.config)}

    # e2e through the public API, headline r: host x -> H2D -> graph -> D2H y
    stack.capture(args.bits)
    gen = torch.Generator().manual_seed(0)
    stack.x_host.copy_(torch.randn(stack.x_host.shape, generator=gen).to(torch.bfloat16))
    for _ in range(args.warmup):
        stack.decode()
    e2e_secs = time_steps(stack.decode, args.steps)
    h2d, d2h = stack.io_bytes()

    # roofline: the dominant kernel, gate_up GEMV, each launch on its own (cold) weights
    gu = [pt for _, kind, pt in stack.layers if kind == "gate_up"]
    r = args.bits
    xg = stack.bufs["o"]
    outg = stack.bufs["gate_up"]
    with torch.cuda.stream(stack.stream):
        for pt in gu:
            pt.gemv(xg, r, out=outg, stream=stack.stream)
    ktimes = []
    for _ in range(3):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stack.stream)
        with torch.cuda.stream(stack.stream):
            for pt in gu:
                pt.gemv(xg, r, out=outg, stream=stack.stream)
        e1.record(stack.stream)
        barrier()
        ktimes.append(e0.elapsed_time(e1) / 1e3 / len(gu))
    k_sec = max_over_ranks(min(ktimes))
    pt0 = gu[0]
    kbytes = algorithmic_bytes(pt0.N, pt0.K, args.batch, r, pt0.planes_read(r), 128)
    achieved = kbytes / k_sec / 1e9
    traffic_db = {}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic_db = json.load(f)
    except Exception:
        pass
    roof_k3 = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
               "traffic": traffic_db.get("k_gemv_gate_up_r%d_b%d" % (r, args.batch)),
               "kernel": "k_gemv gate_up %dx%d r=%d B=%d (per-layer K3)" % (pt0.N, pt0.K, r, args.batch),
               "bytes_per_launch": kbytes, "us_per_launch": k_sec * 1e6, "peak_kind": peak_kind}

    # the headline's dominant kernel: with a uniform config the whole step is one
    # K3S launch (k_stack); time bare launches (no graph) with CUDA events
    stack.capture(r)
    roof = roof_k3
    if stack.program is not None:
        with torch.cuda.stream(stack.stream):
            stack.program.run(stack.stream)
        stimes = []
        for _ in range(3):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stack.stream)
            for _ in range(4):
                stack.program.run(stack.stream)
            e1.record(stack.stream)
            barrier()
            stimes.append(e0.elapsed_time(e1) / 1e3 / 4)
        s_sec = max_over_ranks(min(stimes))
        sbytes = stack.step_bytes(stack.config)
        roof = {"bound": "hbm", "achieved": sbytes / s_sec / 1e9, "peak": peak, "unit": "GB/s",
                "frac": sbytes / s_sec / 1e9 / peak,
                "traffic": traffic_db.get("k_stack_r%d_b%d" % (r, args.batch)),
                "kernel": "k_stack (K3S: the whole %d-layer step, one launch) r=%d B=%d" % (
                    len(stack.layers), r, args.batch),
                "bytes_per_launch": sbytes, "us_per_launch": s_sec * 1e6, "peak_kind": peak_kind}

    # per-layer-kind breakdown: one CUDA graph of the 32 same-kind launches (PDL)
    kinds = {}
    for kind in ("qkv", "o", "gate_up", "down"):
        pts = [pt for _, k2, pt in stack.layers if k2 == kind]
        xin = {"qkv": stack.x, "o": stack.bufs["qkv"][:, :pts[0].K], "gate_up": stack.bufs["o"],
               "down": stack.bufs["gate_up"][:, :pts[0].K]}[kind]
        outk = {"qkv": stack.bufs["qkv"], "o": stack.bufs["o"], "gate_up": stack.bufs["gate_up"],
                "down": stack.x}[kind]
        with torch.cuda.stream(stack.stream):
            for pt in pts:
                pt.gemv(xin, r, out=outk, pdl=True, stream=stack.stream)
        stack.stream.synchronize()
        gk = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gk, stream=stack.stream):
            for pt in pts:
                pt.gemv(xin, r, out=outk, pdl=True, stream=stack.stream)
        with torch.cuda.stream(stack.stream):
            gk.replay()
        def replay_k(g=gk):
            with torch.cuda.stream(stack.stream):
                g.replay()

        secs = time_steps(replay_k, 5) / 5 / len(pts)
        nb = algorithmic_bytes(pts[0].N, pts[0].K, args.batch, r, pts[0].planes_read(r), 128)
        kinds[kind] = {"us": secs * 1e6, "GBps": nb / secs / 1e9, "frac": nb / secs / 1e9 / peak,
                       "N": pts[0].N, "K": pts[0].K}
        del gk

    # mode C (materialised children) for the headline r
    mode_c = None
    if r < 8 and world == 1 and not args.no_sweep:
        saved = [(i, pt) for i, (_, _, pt) in enumerate(stack.layers)]
        try:
            for i, (n, kind, pt) in enumerate(stack.layers):
                stack.layers[i] = (n, kind, pt.materialize_child(r))
            stack.capture(r)
            for _ in range(args.warmup):
                stack.step()
            secs = time_steps(stack.step, args.steps)
            mode_c = args.batch * args.steps / secs
        except torch.cuda.OutOfMemoryError:
            mode_c = None
        finally:
            for i, pt in saved:
                n, kind, _ = stack.layers[i]
                stack.layers[i] = (n, kind, pt)
            torch.cuda.empty_cache()

    # C2: uniform r, decode batch 1-16
    c2 = None
    if not args.no_c2 and world == 1:
        c2 = sweep_leg(torch, stack, clocks, peak, (1, 2, 4, 8, 16), [("r%d" % b, b) for b in LADDER])

    # C3: heterogeneous per-layer bit-widths (EvoPress-style budget-exact 3.5-bit
    # config over the unfused linears, the reference's own moves): the default
    # dispatch -- the per-layer-r K3S kernel at B <= 4, else the per-layer graph
    hetero = None
    if not args.no_hetero and args.model == "Llama-3.1-8B":
        from paper_2602_03537_b200.config import budget_config, level_histogram

        stack.graph = None
        cfg = budget_config(3.5, shape=shape, seed=0, mutations=200, n_layers=args.layers)
        hs = LinearStack(shape, batch=args.batch, tp=world, rank=rank, process_group=pg,
                         n_layers=args.layers, fused=False)
        hs.capture(cfg.assignment)
        for _ in range(args.warmup):
            hs.step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks.active(True)
        e0.record(hs.stream)
        for _ in range(args.steps):
            hs.step()
        e1.record(hs.stream)
        barrier()
        clocks.active(False)
        hsec = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        hb = hs.step_bytes(hs.config)
        hetero = {"tok_s": args.batch * args.steps / hsec, "ms_per_step": hsec / args.steps * 1e3,
                  "avg_bits": 3.5, "histogram": {str(k): v for k, v in level_histogram(cfg).items()},
                  "launches_per_step": hs.launches_per_step(), "GB_per_step": hb / 1e9,
                  "stack_GBps": hb / (hsec / args.steps) / 1e9,
                  "stack_frac": hb / (hsec / args.steps) / 1e9 / peak,
                  "config": "budget_config(3.5, seed=0, mutations=200) over 224 unfused linears"}
        if not args.no_c2:
            hetero["batch_sweep"] = sweep_leg(torch, hs, clocks, peak, (1, 8, 16, 32),
                                              [("hetero3.5", cfg.assignment)])
        del hs
        torch.cuda.empty_cache()

    # Full-model decode (BASELINE C5): the same sliced
    # linears inside Llama-3.1-8B / Qwen3-14B / Phi-3-Medium-shaped decoders
    # (bf16 attention over a 256-token KV cache, RMSNorm, RoPE, SiLU, bf16
    # lm_head), one CUDA graph per token, tensor-parallel over the N ranks
    # (tp.decoder_plan, NCCL all-reduces in the graph); set beside the paper's
    # own full-model numbers (RTX A6000)
    full = None
    if not args.no_full:
        from paper_2602_03537_b200.llama import LlamaDecoder
        from paper_2602_03537_b200.shapes import SHAPES as DSHAPES

        stack.graph = None
        torch.cuda.empty_cache()
        paper = {2: 138.0, 3: 124.4, 4: 109.3}
        vocab = {"Llama-3.1-8B": 128256, "Qwen3-14B": 151936, "Phi-3-Medium": 32064}
        full = {"context": 256, "lm_head": "bf16, replicated", "attention": "torch SDPA (GQA), bf16",
                "tp": world, "models": {}}
        for mname in ("Llama-3.1-8B", "Qwen3-14B", "Phi-3-Medium"):
            dec = LlamaDecoder(DSHAPES[mname], batch=args.batch, context=256, bits=args.bits,
                               vocab=vocab[mname], n_layers=args.layers, tp=world, rank=rank, process_group=pg)
            rec_m = {"per_bits": {}}
            for rb in ((2, 3, 4, 8) if mname == "Llama-3.1-8B" else (args.bits,)):
                dec.set_bits(rb)
                dec.capture()
                for _ in range(args.warmup):
                    dec.step()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                clocks.active(True)
                e0.record(dec.stream)
                for _ in range(args.steps):
                    dec.step()
                e1.record(dec.stream)
                barrier()
                clocks.active(False)
                fsec = max_over_ranks(e0.elapsed_time(e1) / 1e3 / args.steps)
                rec = {"tok_s": args.batch / fsec, "ms_per_step": fsec * 1e3}
                if mname == "Llama-3.1-8B" and rb in paper and args.batch == 1:
                    rec["paper_a6000_tok_s"] = paper[rb]
                    rec["vs_paper"] = (args.batch / fsec) / paper[rb]
                rec_m["per_bits"][str(rb)] = rec
            dec.set_bits(args.bits)
            rec_m["components_ms_r%d" % args.bits] = dec.component_ms()
            full["models"][mname] = rec_m
            del dec
            torch.cuda.empty_cache()

    # C1: one 4096x4096 linear (the reference bench's case), L2-cold
    c1 = None
    if not args.no_c1 and world == 1:
        stack.graph = None
        torch.cuda.empty_cache()
        c1 = c1_leg(torch, mq, clocks, peak, cpu=not args.no_cpu)

    # C4: prefill on the tcgen05 path (K4), Qwen3-14B linear shapes, per layer
    prefill = None
    if not args.no_prefill and world == 1:
        prefill = prefill_leg(torch, mq, clocks)

    # the quantiser's searches
    quant = None
    if not args.no_quant and world == 1:
        quant = quant_leg(torch, mq, cpu=not args.no_cpu)

    clk = clocks.summary()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference as shipped: its compiled kernel on ONE core (_core.pyx:47-63 is
        # single-threaded, matmul.py:164 threadpool_limits(1)); one whole decode step
        ref = CpuReference(r, args.batch, 1, args.model)
        ref.block_seconds()  # warm-up
        secs = ref.step_seconds()
        ref.close()
        cpu = {"value": args.batch / secs, "unit": UNIT, "cores": 1, "kind": ref.kind,
               "host_cores": os.cpu_count(),
               "sample": "one whole decode step (%d blocks x 4 linears, all rows, one block's weights "
                         "reused per block) at r=%d on 1 of %d host cores; %s" % (
                             ref.n_blocks, r, os.cpu_count() or 1, ref.backend)}

    head = results[args.bits]
    bytes_tok = head["bytes_per_step"] * world / args.batch
    line = {
        "metric": METRIC, "value": head["tok_s"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init int8 parents, N(0,1) bf16 activations)",
        "config": workload_config(args.model, n_blocks, args.bits, args.batch, world),
        "run": {"mode": "P (parent resident, sliced on the fly)",
                "l2": "inputs > L2 (%.1f GB of planes read per step vs 126 MB L2)" % (
                    head["bytes_per_step"] / 1e9),
                "graph": ("CUDA graph of 1 K3S launch/step (persistent whole-step kernel)"
                          if head_launches == 1 else
                          "CUDA graph, %d K3 launches/step, PDL" % head_launches)},
        "per_bits": {str(b): {"tok_s": v["tok_s"], "ms_per_step": v["ms_per_step"],
                              "GB_per_step": v["bytes_per_step"] / 1e9,
                              "stack_GBps": v["bytes_per_step"] / (v["ms_per_step"] / 1e3) / 1e9,
                              "stack_frac": v["bytes_per_step"] / (v["ms_per_step"] / 1e3) / 1e9 / peak}
                     for b, v in results.items()},
        "mode_c_tok_s": mode_c,
        "per_kind_r%d" % args.bits: kinds,
        "bytes_per_token": bytes_tok,
        "e2e": {"value": args.batch * args.steps / e2e_secs, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": roof,
        "roofline_k3_gate_up": roof_k3,
        "full_model_decode": full,
        "c1_single_linear": c1,
        "c2_batch_sweep": c2,
        "hetero_c3": hetero,
        "prefill_c4": prefill,
        "quantizer_8f4": quant,
        "cpu_baseline": cpu,
        "clocks": clk,
        # K3 launches inside the headline timed region (K captured steps)
        "gpu_launches": head_launches * args.steps,
        "backend": mq.kernels.backend_name(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
