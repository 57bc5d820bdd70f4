cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x --timeout 300 2>&1 | tail -30
