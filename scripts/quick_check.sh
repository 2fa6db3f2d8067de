timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
SHAPES=gate_up,down BITS=2,4,8 WARPS=16 STAGES=3 SPLITS=0 timeout 300 python scripts/sweep_gemv.py > gpurun_out/sweep.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
