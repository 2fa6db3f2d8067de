#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stack.py -q -x -p no:cacheprovider -k "gemv or stack or forced or split or golden or c1" 2>&1 | tail -2
for b in 4 8 16 32; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-hetero --no-prefill --no-sweep --batch $b > gpurun_out/bb_$b.json 2> gpurun_out/bb_$b.err
  python - gpurun_out/bb_$b.json $b <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("B=%s tok/s %8.1f ms/step %.3f frac %.3f %s" % (sys.argv[2], d["value"], d["ms_per_step"], d["roofline"]["frac"], json.dumps({k: round(v["us"], 1) for k, v in d["per_kind_r4"].items()})))
PY
done
