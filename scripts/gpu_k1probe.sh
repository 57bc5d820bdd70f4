mkdir -p gpurun_out
for L in "" paper_2503_16672_b200/_exp/libs24_k1p1.so paper_2503_16672_b200/_exp/libs24_k1p2.so; do
  echo "== lib [$L]"; S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep "K1\|relu2\|fwd.out dense"
done
timeout 300 python scripts/k4_only.py > /dev/null 2>&1; echo k4only rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_feature_split -s 2 -c 1 -o gpurun_out/prof_k4d python scripts/k4_only.py > gpurun_out/ncu_k4d.log 2>&1; echo rc=$?
