#!/bin/bash
# K3 A/B: full GPU suite on the default build, then the heterogeneous matrix rows and the
# full-model decode leg for A (default) and B ($1).
mkdir -p gpurun_out; rm -f gpurun_out/ab_k3.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for v in A B; do
  if [ $v = B ]; then export MQ_LIB_PATH=$1; else unset MQ_LIB_PATH; fi
  echo "== $v" >> gpurun_out/ab_k3.txt
  PYTHONPATH=. timeout 600 python scripts/stack_matrix.py 1 h 2>/dev/null | grep -v Warn >> gpurun_out/ab_k3.txt
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-prefill --no-hetero --no-quant --no-sweep > gpurun_out/abk3_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/abk3_$v.json').read().strip().splitlines()[-1])
print('full', {k:round(v['tok_s'],1) for k,v in d['full_model_decode']['per_bits'].items()}, 'kinds', {k: round(v['us'],1) for k,v in d['per_kind_r4'].items()})" >> gpurun_out/ab_k3.txt
done
