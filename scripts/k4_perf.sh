#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/bench_prefill.py > gpurun_out/prefill.jsonl 2> gpurun_out/prefill.err
tail -3 gpurun_out/prefill.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 -o gpurun_out/prof_k4_gateup_b512_r4 python scripts/prof_gemm.py 34816 5120 4 512 > gpurun_out/ncu_k4.log 2>&1
tail -3 gpurun_out/ncu_k4.log
