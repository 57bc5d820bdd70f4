cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo c2 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/final_c2.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','eager_ms_per_step','speedup_vs_dense','sparse_tflops','gpu_launches')}); print(' dense', d.get('dense_twin')); print(' fp8', d.get('fp8_variant')); print(' roof', {k: d['roofline'][k] for k in ('kernel','achieved','peak','frac')}); print(' clocks', d['clocks'])"
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense --no-fp8"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv $B > /dev/null 2>&1; echo launches rc=$?
