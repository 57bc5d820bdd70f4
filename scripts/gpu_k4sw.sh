S24_LIB=paper_2503_16672_b200/_exp/libs24_k4sw8.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 -k "feature_split or split_weight" 2>&1 | tail -1
for L in "" paper_2503_16672_b200/_exp/libs24_k4sw4.so paper_2503_16672_b200/_exp/libs24_k4sw8.so paper_2503_16672_b200/_exp/libs24_k4sw16.so; do
  echo "== [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep "K4x\|K4 feature"
done
