#!/bin/bash
# K3 decomposition variants: does PDL co-residency (<= half-SM CTAs) pay?
mkdir -p gpurun_out
for v in "16 0" "8 3" "8 2" "16 2" "4 3"; do
  set -- $v
  if [ "$2" = 0 ]; then st=""; else st="MQ_GEMV_STAGES=$2"; fi
  env MQ_GEMV_WARPS=$1 $st timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-sweep > gpurun_out/var_w$1_s$2.json 2> gpurun_out/var_w$1_s$2.err
  python - gpurun_out/var_w$1_s$2.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=d["per_kind_r4"]
print(sys.argv[1], "tok/s %.1f" % d["value"], " ".join("%s %.2fus %.2f" % (n, v["us"], v["frac"]) for n, v in k.items()))
PY
done
