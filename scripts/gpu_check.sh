# GPU tests + bench line (+ kernel breakdown)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_check.json 2>gpurun_out/bench_check.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_check.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], "eager", d.get("eager_ms_per_step"), "speedup", d.get("speedup_vs_dense"), "dense", (d.get("dense_twin") or {}).get("ms_per_step"), "e2e", d.get("e2e",{}).get("value"), d["clocks"], d.get("cpu_baseline"))
for k in d["kernels"]: print("   ", k["kernel"], round(k["ms_per_step"],4), k["launches_per_step"])
PY
