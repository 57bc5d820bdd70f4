mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -4
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/b_pair.json 2>gpurun_out/b_pair.err; echo rc=$?
S24_PAIRED_WGRAD=0 timeout 300 python bench.py --no-cpu --no-e2e --no-dense > gpurun_out/b_nopair.json 2>&1; echo rc=$?
python - <<'PY'
import json
for f in ["gpurun_out/b_pair.json","gpurun_out/b_nopair.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, e); continue
    print(f, d["ms_per_step"], d.get("speedup_vs_dense"), (d.get("dense_twin") or {}).get("ms_per_step"))
    for k in d["kernels"]: print("   ", k["kernel"], round(k["ms_per_step"],4), k["launches_per_step"])
PY
