timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -3
timeout 900 python bench.py --config c3 --steps 5 --no-cpu > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config c4 --steps 5 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; echo c4 rc=$?
python - <<'PY'
import json
for f in ["gpurun_out/bench_c3.json", "gpurun_out/bench_c4.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["config"]["workload"], d["ms_per_step"], d.get("speedup_vs_dense"), d["sparse_tflops"], d.get("e2e", {}).get("value"), d["drops"])
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-1500:])
PY
