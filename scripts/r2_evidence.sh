# Round-2 evidence: GPU suite, smoke, bench line (+ reference arm), the bench's ncu
# launch list, one full ncu capture of the K3S step, the C4 prefill sweep
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python scripts/prefill_graph.py 64,128,256,512,1024 4,8 > gpurun_out/prefill_graph.txt 2>&1; echo "prefill rc=$?"
MQ_STACK_NOCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --kernel-name regex:"k_stack|k_gemv|k_gemm|k_add_rmsnorm|k_rope_kv|k_silu_mul" \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-c2 --no-full --no-prefill --no-quant --no-cpu --no-hetero --no-c1 > gpurun_out/launch_bench.log 2>&1; echo "launches rc=$?"
MQ_STACK_NOCOOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stack -s 1 -c 1 \
  -o gpurun_out/r2_k3s_final python scripts/prof_stack.py 4 1 32 > gpurun_out/r2_k3s_final.log 2>&1; echo "ncu rc=$?"
