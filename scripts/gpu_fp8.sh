cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_ffn_fp8.py -q --timeout 600 2>&1 | grep -E "^(FAILED|E  )" | head -40
