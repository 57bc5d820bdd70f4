#!/bin/bash
# wide dense tiles: parity, then per-kernel timing narrow vs wide
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ffn.py tests/test_gpu_fp8.py tests/test_gpu_ffn_fp8.py -x -q -m gpu 2>&1 | tail -5
for bn in 256 512 256 512; do
  echo "== S24_DENSE_BN=$bn"
  S24_DENSE_BN=$bn python scripts/kernel_bench.py --config c2 --iters 20 2>&1 | grep -E "K1|relu2|plain|dense twin|K3|dact"
done
