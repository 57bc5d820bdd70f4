for L in "" paper_2503_16672_b200/_exp/libs24_probe3.so paper_2503_16672_b200/_exp/libs24_probe1.so; do
  echo "== lib [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep -v "K7\|K4\|K6" | cut -c1-90
done
