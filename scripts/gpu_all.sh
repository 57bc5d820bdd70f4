cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -15
timeout 300 python -m pytest tests/test_gpu_ffn_fp8.py -q -s --timeout 300 2>&1 | grep reported
