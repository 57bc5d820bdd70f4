#!/bin/bash
# recipe step time for each K4 placement (and the fused-epilogue variant)
for mode in side inline background; do
  S24_K4_MODE=$mode timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>&1 | tail -1 > gpurun_out/b_$mode.json
done
S24_FUSED_FW=1 timeout 300 python bench.py --steps 10 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/b_fused.json
for f in side inline background fused; do python -c "
import json
d=json.load(open('gpurun_out/b_$f.json'))
print('$f', round(d['ms_per_step'],4), d.get('dense_twin',{}).get('ms_per_step'))
for k in d['kernels']: print('  ', round(k['ms_per_step'],4), round(k['frac'] or 0,3), k['kernel'])
"; done
