cd $GRAFT_REPO_ROOT
for r in 1 2; do
for L in paper_2503_16672_b200/libs24.so paper_2503_16672_b200/_exp/libs24_pf4.so paper_2503_16672_b200/_exp/libs24_pf8.so paper_2503_16672_b200/_exp/libs24_pf16.so; do echo $L; S24_LIB=$L timeout 300 python scripts/kernel_bench.py --config c2 --iters 10 2>&1 | grep -E "sparse" | cut -c1-70; done
done
