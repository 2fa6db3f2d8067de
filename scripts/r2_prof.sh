# K3S evidence: per-layer phase timeline (timing build) + one ncu capture with source counters
mkdir -p gpurun_out
for r in 4 2; do MQ_LIB_PATH=build/timing/libmatq.so timeout 200 python scripts/stack_timing.py $r 1 32 2>&1 | grep -v k_stack; done
MQ_STACK_NOCOOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stack -s 1 -c 1 -o gpurun_out/${1:-r2_k3s} python scripts/prof_stack.py 4 1 8 > gpurun_out/${1:-r2_k3s}.log 2>&1; tail -2 gpurun_out/${1:-r2_k3s}.log
