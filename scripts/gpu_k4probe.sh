for L in "" paper_2503_16672_b200/_exp/libs24_k4p1.so paper_2503_16672_b200/_exp/libs24_k4p2.so; do
  echo "== [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep "K4x"
done
