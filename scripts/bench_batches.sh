#!/bin/bash
# Decode batch sweep (BASELINE config: batch 1-16, plus 32): headline bench legs only.
mkdir -p gpurun_out; rm -f gpurun_out/batches.txt
for b in 1 2 4 8 16 32; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-hetero --no-prefill --no-quant --no-full --no-sweep --batch $b > gpurun_out/bb_$b.json 2> gpurun_out/bb_$b.err
  python - gpurun_out/bb_$b.json $b >> gpurun_out/batches.txt <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("B=%s r=4 tok/s %8.1f ms/step %.3f stack GB/s %.0f frac %.3f | %s" % (sys.argv[2], d["value"], d["ms_per_step"], d["per_bits"]["4"]["stack_GBps"], d["per_bits"]["4"]["stack_frac"], d["config"]["graph"]))
PY
done
