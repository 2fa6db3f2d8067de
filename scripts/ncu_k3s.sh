#!/bin/bash
# Full ncu capture of the headline K3S launch (r=4, B=1, Llama-3.1-8B stack) + a launch check.
mkdir -p gpurun_out
MQ_STACK_LAUNCH_DEBUG=1 timeout 300 python scripts/prof_stack.py 4 1 32 > gpurun_out/k3s_plain.log 2>&1; echo rc=$? >> gpurun_out/k3s_plain.log
MQ_STACK_LAUNCH_DEBUG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stack -s 1 -c 1 -o gpurun_out/prof_k3s_full python scripts/prof_stack.py 4 1 32 > gpurun_out/ncu_k3s_full.log 2>&1; echo rc=$? >> gpurun_out/ncu_k3s_full.log
