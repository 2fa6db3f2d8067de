# ncu evidence: full capture of the gate_up GEMV (r=4 and r=2) + launch list of a short stack bench
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 2 -c 1 -o gpurun_out/prof_gateup_r4 python scripts/prof_one.py 28672 4096 4 1 > gpurun_out/ncu_r4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 2 -c 1 -o gpurun_out/prof_gateup_r2 python scripts/prof_one.py 28672 4096 2 1 > gpurun_out/ncu_r2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gemv --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --layers 2 --no-sweep --no-cpu > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out
