# K3S per-layer phase timeline (timing build) + the GPU API tests + a full bench line
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_api.py -q > gpurun_out/api.log 2>&1; tail -2 gpurun_out/api.log
for r in 4 2; do MQ_LIB_PATH=build/timing/libmatq.so timeout 200 python scripts/stack_timing.py $r 1 32 2>&1 | grep -v k_stack; done > gpurun_out/timing.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
