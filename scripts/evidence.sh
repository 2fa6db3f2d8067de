#!/bin/bash
# Round evidence: GPU tests, smoke, default bench, ncu launch list of the bench, and a
# full ncu capture of the headline kernel (K3S) for the DRAM-traffic figure.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -1 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-hetero --no-prefill --no-quant --no-full > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stack -s 1 -c 1 -o gpurun_out/prof_k3s_full python scripts/prof_stack.py 4 1 32 > gpurun_out/ncu_k3s_full.log 2>&1
ls -la gpurun_out | tail -20
