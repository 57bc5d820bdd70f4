cd $GRAFT_REPO_ROOT
S24_LIB=paper_2503_16672_b200/_exp/libs24_fs8.so timeout 400 python -m pytest tests/test_gpu_ffn.py -q --timeout 300 -k "k4_in_gemm" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -5
S24_LIB=paper_2503_16672_b200/_exp/libs24_fs8.so timeout 900 python scripts/ab_step.py --variants graph,k4_gemm_graph --blocks 6 --steps 5 2>&1 | tail -1
