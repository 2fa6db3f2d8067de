# A/B of libmatq builds on the K3S headline (build/<v>/libmatq.so; "main" = the package's)
for v in ${@:-main old}; do
  if [ $v = main ]; then L=""; else L="MQ_LIB_PATH=build/$v/libmatq.so"; fi
  echo "== $v"; env $L timeout 300 python scripts/k3s_quick.py 1 2 4 8 2>&1 | grep -v k_stack
done
