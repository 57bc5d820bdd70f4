#!/bin/bash
# bench the recipe with the standalone K4 and with K4 fused into the K1/K3 epilogues
python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/b_unfused.json
S24_FUSED_FW=1 python bench.py --steps 10 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/b_fused.json
for f in gpurun_out/b_unfused.json gpurun_out/b_fused.json; do python -c "
import json,sys
d=json.load(open('$f'))
print('$f', d['ms_per_step'], d.get('dense_twin',{}).get('ms_per_step'), d.get('speedup_vs_dense'))
for k in d['kernels']: print('  ', round(k['ms_per_step'],4), round(k['frac'] or 0,3), k['kernel'])
"; done
