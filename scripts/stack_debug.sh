mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stack.py -q -p no:cacheprovider --timeout 120 > gpurun_out/pytest_stack.log 2>&1; echo rc=$? >> gpurun_out/pytest_stack.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-prefill --no-hetero --no-full > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo rc=$? >> gpurun_out/bench_a.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-prefill --no-full > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo rc=$? >> gpurun_out/bench_b.err
