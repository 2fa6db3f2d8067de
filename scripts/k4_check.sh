#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gemm or linear" > gpurun_out/k4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k4_pytest.log
tail -30 gpurun_out/k4_pytest.log
