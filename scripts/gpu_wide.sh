W=paper_2503_16672_b200/_exp/libs24_wide.so
S24_LIB=$W timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 120 -k "spmm or split_weight" 2>&1 | tail -15
S24_LIB=$W timeout 600 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 2>&1 | tail -3
for L in "" $W; do echo "== [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep "sparse" | cut -c1-110; done
