cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','speedup_vs_dense','sparse_tflops')}); print(d.get('dense_twin')); print(d.get('fp8_variant')); print(d['clocks'])"
