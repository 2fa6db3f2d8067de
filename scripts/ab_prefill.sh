#!/bin/bash
# A/B two libmatq builds on the K4 prefill sweep (r=4): $1 = alternative .so (B).
mkdir -p gpurun_out; rm -f gpurun_out/ab_prefill.txt
for v in A B; do
  if [ $v = B ]; then export MQ_LIB_PATH=$1; else unset MQ_LIB_PATH; fi
  echo "== $v" >> gpurun_out/ab_prefill.txt
  timeout 600 python scripts/bench_prefill.py --reps 20 --bits 4 --batches 64,256,1024 2>/dev/null >> gpurun_out/ab_prefill.txt
done
