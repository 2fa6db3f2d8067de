#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/b8.txt
for pair in 1; do for b in 1 2 4 8 16; do
  MQ_STACK_PAIR=$pair timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-hetero --no-prefill --no-quant --no-full --batch $b > gpurun_out/b8_$b.json 2>/dev/null
  python - gpurun_out/b8_$b.json $b $pair >> gpurun_out/b8.txt <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("pair=%s B=%s" % (sys.argv[3], sys.argv[2]), {k: round(v["ms_per_step"], 3) for k, v in d["per_bits"].items()})
PY
done; done
