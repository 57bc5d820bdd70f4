#!/bin/bash
# ncu side-by-side of our dense GEMM and cuBLAS at the K1 shape
set -x
python scripts/dense_vs_cublas.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:'gemm|nvjet|cutlass|sm100' -s 4 -c 2 \
  -o gpurun_out/dense_cmp -f python scripts/dense_vs_cublas.py > gpurun_out/dense_ncu.log 2>&1
ncu -i gpurun_out/dense_cmp.ncu-rep --page details --csv > gpurun_out/dense_cmp_details.csv 2>&1
ncu -i gpurun_out/dense_cmp.ncu-rep --page raw --csv > gpurun_out/dense_cmp_raw.csv 2>&1
tail -3 gpurun_out/dense_ncu.log
