cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_ffn_fp8.py tests/test_gpu_ffn.py -q --timeout 600 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -40
timeout 300 python -m pytest tests/test_gpu_ffn_fp8.py -q -s --timeout 300 2>&1 | grep reported
timeout 900 python scripts/fp8_step.py --config c2 2>&1 | tail -20
