cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ffn.py tests/test_gpu_ffn_fp8.py tests/test_gpu_dp.py -q --timeout 500 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -10
timeout 600 python scripts/kernel_bench.py --config c2 --iters 10 2>&1 | grep -i "K4x"
timeout 900 python scripts/ab_step.py --variants graph,k4_none_graph --blocks 6 --steps 5 2>&1 | tail -1
