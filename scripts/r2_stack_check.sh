mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_stack_parity.py -x -q > gpurun_out/stack_tests.log 2>&1; tail -3 gpurun_out/stack_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python scripts/k3s_quick.py 1 2 3 4 6 8 2>&1 | grep -v "^$" | tail -5
