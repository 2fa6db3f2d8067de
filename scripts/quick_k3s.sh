#!/bin/bash
# K3S A/B loop: stack parity tests + the per-bit-width bench legs only.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stack.py -x -q -p no:cacheprovider > gpurun_out/pytest_stack.log 2>&1; echo rc=$? >> gpurun_out/pytest_stack.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-prefill --no-full --no-hetero --no-quant > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo rc=$? >> gpurun_out/bench_q.err
