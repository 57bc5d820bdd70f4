timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 2>&1 | tail -1
for i in 1 2; do
for L in "" paper_2503_16672_b200/_exp/libs24_nopol.so; do
  echo "== lib [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep -v "K7\|K4\|K6" | cut -c1-100
  S24_LIB=$L timeout 300 python scripts/ab_step.py --blocks 3 --variants graph 2>&1 | tail -1 | cut -c1-80
done
done
