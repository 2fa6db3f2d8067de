# bench the stack with the default GEMV config and with 8-warp CTAs (PDL co-residency)
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-sweep > gpurun_out/bench_w16.json 2> gpurun_out/bench_w16.err
MQ_GEMV_WARPS=8 timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-sweep > gpurun_out/bench_w8.json 2> gpurun_out/bench_w8.err
MQ_GEMV_WARPS=8 MQ_GEMV_STAGES=3 timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-sweep > gpurun_out/bench_w8s3.json 2> gpurun_out/bench_w8s3.err
tail -2 gpurun_out/bench_w16.err
