#!/bin/bash
# final validation of the round: GPU tests, smoke, default bench, c3/c4 lines, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo c2 rc=$?
timeout 900 python bench.py --config c4 --no-e2e --no-cpu > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo c4 rc=$?
timeout 900 python bench.py --config c3 --no-e2e --no-cpu > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; echo c3 rc=$?
for c in c2 c4 c3; do python -c "
import json,sys; d=json.loads(open('gpurun_out/final_$c.json').read().strip().splitlines()[-1])
print('$c', {k: d.get(k) for k in ('value','ms_per_step','speedup_vs_dense')}, 'dense', (d.get('dense_twin') or {}).get('ms_per_step'), 'fp8', (d.get('fp8_variant') or {}).get('ms_per_step'), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense --no-fp8"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv $B > /dev/null 2>&1; echo launches rc=$?
