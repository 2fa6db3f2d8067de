for w in 16 24 32; do
  lib=""; [ $w != 16 ] && lib="MQ_LIB_PATH=$PWD/build/libmatq_w$w.so"
  env $lib SHAPES=gate_up,down BITS=2,4,8 WARPS=$w STAGES=2,3 SPLITS=0 timeout 300 python scripts/sweep_gemv.py 2>&1 | grep layer
done
