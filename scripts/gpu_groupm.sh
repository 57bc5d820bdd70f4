for G in 1 2 3 2 1; do
  echo "== group_m $G"; S24_GROUP_M=$G timeout 300 python scripts/kernel_bench.py 2>&1 | grep "K1 fwd\|plain\|K3 bwd\|K2\|sparse part\|twin" | cut -c1-90
done
