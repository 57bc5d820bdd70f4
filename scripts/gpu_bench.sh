cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','eager_ms_per_step','speedup_vs_dense','sparse_tflops','gpu_launches')})
print(d.get('fp8_variant')); print(d['roofline']); print(d['e2e']); print(d.get('cpu_baseline')); print(d['clocks'])"
