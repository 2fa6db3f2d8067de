SHAPES=gate_up,down,qkv BITS=4 WARPS=16 STAGES=3 SPLITS=0 STREAMS=0,1 COPIES=8 timeout 300 python scripts/sweep_gemv.py > gpurun_out/sweep.log 2>&1
MQ_GEMV_STREAM=1 timeout 300 ncu --set full --clock-control none -k regex:k_gemv -s 2 -c 1 -o gpurun_out/prof_stream python scripts/prof_one.py 28672 4096 4 1 > gpurun_out/ncu_stream.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "forced or shared or split" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
