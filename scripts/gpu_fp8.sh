cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_ffn_fp8.py tests/test_gpu_dp.py -q --timeout 600 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
timeout 900 python scripts/fp8_step.py --config c2 --rounds 3 2>&1 | head -1
