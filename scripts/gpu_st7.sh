timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 2>&1 | tail -1
S24_LIB=paper_2503_16672_b200/_exp/libs24_st7.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 2>&1 | tail -1
for i in 1 2; do
for L in "" paper_2503_16672_b200/_exp/libs24_st7.so; do
  echo "== lib [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep -v "K7\|K4\|K6\|sparse" | cut -c1-90
done
done
