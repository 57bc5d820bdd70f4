cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ffn.py -q --timeout 500 -k "feature_split or recipe or graph" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -5
for L in paper_2503_16672_b200/_exp/libs24_pipe1.so paper_2503_16672_b200/libs24.so paper_2503_16672_b200/_exp/libs24_pipe4.so; do echo $L; S24_LIB=$L timeout 300 python scripts/kernel_bench.py --config c2 --iters 10 2>&1 | grep -i "K4x"; done
timeout 600 python scripts/ab_step.py --variants graph,k4_none_graph --blocks 6 --steps 5 2>&1 | tail -1
