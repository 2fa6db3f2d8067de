# A/B of libmatq builds (build/<v>/libmatq.so) on the K3S headline: k3s_quick per width
for v in "$@"; do
  echo "== $v"; MQ_LIB_PATH=build/$v/libmatq.so timeout 300 python scripts/k3s_quick.py 1 ${WIDTHS:-2 4 8} 2>&1 | grep "r="
done
