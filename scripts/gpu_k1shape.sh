mkdir -p gpurun_out
timeout 300 python scripts/kernel_bench.py 2>&1 | grep "K1\|relu2\|plain\|K3\|dact"
timeout 300 python scripts/gemm_only.py k1 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_k1c python scripts/gemm_only.py k1 > gpurun_out/ncu_k1c.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_relu2c python scripts/gemm_only.py relu2 > gpurun_out/ncu_relu2c.log 2>&1; echo rc=$?
