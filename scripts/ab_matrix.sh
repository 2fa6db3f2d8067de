#!/bin/bash
# A/B two libmatq builds on scripts/stack_matrix.py (heterogeneous rows): $1 = alternative .so (B).
mkdir -p gpurun_out; rm -f gpurun_out/ab_matrix.txt
for v in A B; do
  if [ $v = B ]; then export MQ_LIB_PATH=$1; else unset MQ_LIB_PATH; fi
  echo "== $v" >> gpurun_out/ab_matrix.txt
  PYTHONPATH=. timeout 600 python scripts/stack_matrix.py 1 h 2>/dev/null | grep -v Warn >> gpurun_out/ab_matrix.txt
done
