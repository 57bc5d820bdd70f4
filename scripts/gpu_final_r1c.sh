#!/bin/bash
# end-of-session validation: GPU tests, smoke, default bench (c2), fp8 step launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final2_c2.json 2> gpurun_out/final2_c2.err; echo c2 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/final2_c2.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','speedup_vs_dense')}, 'dense', d['dense_twin']['ms_per_step'], 'fp8', d['fp8_variant']['ms_per_step'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), 'frac', d['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_fp8_c2_v2.csv python scripts/fp8_prof.py > /dev/null 2>&1; echo launches rc=$?
python scripts/launch_summary.py gpurun_out/launches_fp8_c2_v2.csv > gpurun_out/launches_fp8_c2_v2.txt 2>&1; head -40 gpurun_out/launches_fp8_c2_v2.txt
