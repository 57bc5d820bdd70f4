mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 120 2>&1 | tail -5
S24_LIB=paper_2503_16672_b200/_exp/libs24_dmc2.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 120 2>&1 | tail -5
for L in "" paper_2503_16672_b200/_exp/libs24_smc1.so paper_2503_16672_b200/_exp/libs24_dmc2.so; do
  echo "== lib $L"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | tail -14
done
