for m in 0 1 2; do echo "MQ_SHR_MODE=$m"; timeout 100 ./scripts/micro/decode_rate_m$m | grep "warps=16"; done
