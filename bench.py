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


# ------------------------------------------------------------ CPU baseline --
class CpuReference:
    """One Llama-3.1-8B block (qkv, o, gate_up, down) on the host cores.

    r in {2,3,4}: the reference's compiled nq_gemv/nq_gemm (oracle/_ref, driven
    as kernels/_core.pyx:24-64 drives it), rows spread over `threads` host
    threads (the kernel walks rows independently, packed_kernels.c:88; ctypes
    releases the GIL).  r in {6,8}: the reference has no packed kernel
    (matmul.py:55-56); its bench baseline, a dense fp32 GEMV on the
    dequantised child (matmul.py:164-165), is used instead.
    Preparation (slice + pack) is untimed, as in the reference bench.
    """

    def __init__(self, r: int, batch: int, threads: int):
        import numpy as np
        from concurrent.futures import ThreadPoolExecutor

        from oracle import oracle as O
        from paper_2602_03537_b200.model import KINDS, LLAMA31_8B, tp_layer_dims

        self.r, self.threads, self.O = r, threads, O
        rng = np.random.default_rng(0)
        self.layers = []
        for kind in KINDS:
            N, K = tp_layer_dims(LLAMA31_8B, kind, 1)
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
        self.pool = ThreadPoolExecutor(max_workers=threads)
        self.kind = "reference" if r <= 4 else "port"
        self.backend = (self.ref.backend_name() if self.ref
                        else "dense-fp32 GEMV (oracle C; the reference bench's baseline)")

    def _layer(self, ly):
        kind, N = ly[0], ly[1]
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

    def close(self):
        self.pool.shutdown()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    r = args.bits
    ref = CpuReference(r, args.batch, threads)
    samples = []
    for i in range(args.warmup + args.steps):
        t = ref.block_seconds()
        if i >= args.warmup:
            samples.append(t)
    ref.close()
    kind, backend = ref.kind, ref.backend
    per_block = statistics.median(samples)
    tok_s = args.batch / (32 * per_block)
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 32 * per_block * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic",
        "config": {"workload": "Llama-3.1-8B linear stack decode (32 blocks x qkv/o/gate_up/down), "
                               "int8 parent sliced to r=%d, G=128" % r,
                   "model": "Llama-3.1-8B", "bits": r, "batch": args.batch, "group_size": 128},
        "cpu_baseline": {"value": tok_s, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": "one full transformer block (4 linears, all rows) per step, "
                                   "x32 blocks; backend %s" % backend},
        "e2e": {"value": tok_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="matq", choices=["matq", "reference"])
    ap.add_argument("--bits", type=int, default=4, choices=LADDER)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=None, help="debug: fewer blocks")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
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
    from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack

    peak, peak_kind = _peaks()
    stack = LinearStack(LLAMA31_8B, batch=args.batch, tp=world, rank=rank, process_group=pg,
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
    for r in order:
        stack.capture(r)
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
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("gate_up_r%d_b%d" % (r, args.batch))
    except Exception:
        pass

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

    clk = clocks.summary()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        ref = CpuReference(r, args.batch, threads)
        ref.block_seconds()  # warm-up
        per_block = statistics.median(ref.block_seconds() for _ in range(3))
        ref.close()
        cpu = {"value": args.batch / (32 * per_block), "unit": UNIT, "cores": threads,
               "kind": ref.kind,
               "sample": "one full Llama-3.1-8B block (4 linears, all rows) at r=%d, median of 3, "
                         "x32 blocks; %s" % (r, ref.backend)}

    head = results[args.bits]
    bytes_tok = head["bytes_per_step"] * world / args.batch
    line = {
        "metric": METRIC, "value": head["tok_s"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init int8 parents, N(0,1) bf16 activations)",
        "config": {"workload": "Llama-3.1-8B linear stack decode: %d blocks x {qkv 6144x4096, "
                               "o 4096x4096, gate_up 28672x4096, down 4096x14336}, int8 parent "
                               "sliced on the fly (mode P), G=128" % n_blocks,
                   "model": "Llama-3.1-8B", "bits": args.bits, "batch": args.batch,
                   "group_size": 128, "parallelism": "tp%d" % world,
                   "l2": "inputs > L2 (%.1f GB of planes read per step vs 126 MB L2)" % (
                       head["bytes_per_step"] / 1e9),
                   "graph": "CUDA graph, %d K3 launches/step, PDL" % stack.launches_per_step()},
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
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_gemv gate_up %dx%d r=%d B=%d" % (pt0.N, pt0.K, r, args.batch),
                     "bytes_per_launch": kbytes, "us_per_launch": k_sec * 1e6,
                     "peak_kind": peak_kind},
        "cpu_baseline": cpu,
        "clocks": clk,
        # K3 launches inside the headline timed region (K captured steps)
        "gpu_launches": stack.launches_per_step() * args.steps,
        "backend": mq.kernels.backend_name(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
