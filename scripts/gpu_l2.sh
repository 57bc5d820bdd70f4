mkdir -p gpurun_out
for L in "" paper_2503_16672_b200/_exp/libs24_cs.so paper_2503_16672_b200/_exp/libs24_hint.so paper_2503_16672_b200/_exp/libs24_cshint.so; do
  echo "== lib [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep -v "K7\|K4\|K6" | cut -c1-110
  S24_LIB=$L timeout 300 python scripts/ab_step.py --blocks 4 --variants default 2>&1 | tail -1
done
