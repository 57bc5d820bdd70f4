cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q --timeout 600 -k feature_split 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
timeout 600 python scripts/kernel_bench.py --config c2 --iters 10 2>&1 | grep -i "K4x"
