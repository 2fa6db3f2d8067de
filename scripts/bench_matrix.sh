#!/bin/bash
# BASELINE configs C2/C5 on one GPU: batch sweep and the other model shapes (headline leg only)
mkdir -p gpurun_out
for args in "--batch 4" "--batch 16" "--batch 32" "--model Qwen3-14B" "--model Phi-3-Medium" "--bits 2" "--bits 8"; do
  tag=$(echo $args | tr ' ' '_' | tr -d '-')
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-hetero --no-prefill --no-sweep $args > gpurun_out/bm_$tag.json 2> gpurun_out/bm_$tag.err
  python - gpurun_out/bm_$tag.json "$args" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("%-22s tok/s %8.1f  e2e %8.1f  frac %.3f  %s" % (sys.argv[2], d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["config"]["graph"]))
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
