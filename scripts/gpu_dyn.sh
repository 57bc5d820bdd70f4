mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -4
for L in "" paper_2503_16672_b200/_exp/libs24_static.so; do
  echo "== lib $L"
  S24_LIB=$L timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/b_dyn.json 2>gpurun_out/b_dyn.err; echo rc=$?
  python - <<'PY'
import json
d=json.loads(open("gpurun_out/b_dyn.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d.get("speedup_vs_dense"), (d.get("dense_twin") or {}).get("ms_per_step"))
for k in d["kernels"]: print("   ", k["kernel"], round(k["ms_per_step"],4), k["launches_per_step"])
PY
  S24_LIB=$L timeout 300 python scripts/kernel_bench.py 2>&1 | grep -v "K7\|K4\|K6"
done
