cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo c2 rc=$?
timeout 900 python bench.py --config c3 --steps 5 > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; echo c3 rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref rc=$?
for f in final_c2 final_c3; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', {k: d.get(k) for k in ('value','ms_per_step','eager_ms_per_step','speedup_vs_dense','sparse_tflops','gpu_launches')}); print(' dense', d.get('dense_twin')); print(' fp8', d.get('fp8_variant')); print(' roof', {k: d['roofline'][k] for k in ('kernel','achieved','peak','frac')}); print(' e2e', d.get('e2e',{}).get('value')); print(' clocks', d['clocks'])"; done
tail -1 gpurun_out/final_ref.json | cut -c1-400
