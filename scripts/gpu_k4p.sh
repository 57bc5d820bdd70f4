cd $GRAFT_REPO_ROOT
for L in paper_2503_16672_b200/libs24.so paper_2503_16672_b200/_exp/libs24_minb5.so paper_2503_16672_b200/_exp/libs24_minb6.so paper_2503_16672_b200/libs24.so; do echo $L; S24_LIB=$L timeout 300 python scripts/kernel_bench.py --config c2 --iters 10 2>&1 | grep -i "K4x"; done
