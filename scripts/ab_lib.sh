#!/bin/bash
# A/B two libmatq builds on the per-bit-width K3S bench: $1 = alternative .so (B), default build = A.
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for v in A B A B; do
  if [ $v = B ]; then export MQ_LIB_PATH=$1; else unset MQ_LIB_PATH; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-prefill --no-full --no-hetero --no-quant > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
print('$v', {k:round(v['tok_s'],1) for k,v in d['per_bits'].items()})" >> gpurun_out/ab.txt
done
