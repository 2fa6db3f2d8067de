#!/bin/bash
# ncu full captures of the two large Llama GEMVs (steady-state streaming)
mkdir -p gpurun_out
for s in "28672 4096 4" "4096 14336 4" "28672 4096 2" "4096 4096 4"; do
  set -- $s
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 3 -c 1 \
     -o gpurun_out/prof_${1}x${2}_r$3 python scripts/prof_one.py $1 $2 $3 1 6 > gpurun_out/ncu_${1}x${2}_r$3.log 2>&1
done
ls gpurun_out
