# Round-2 GPU evidence: the GPU suite, smoke, and one ncu capture of the K3S step
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ "${PROF:-1}" = 1 ]; then
MQ_STACK_NOCOOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stack -s 1 -c 1 \
  -o gpurun_out/${TAG:-r2_k3s} python scripts/prof_stack.py 4 1 32 > gpurun_out/${TAG:-r2_k3s}.log 2>&1
tail -3 gpurun_out/${TAG:-r2_k3s}.log
fi
