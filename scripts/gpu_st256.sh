#!/bin/bash
# 256-bit epilogue stores: parity, per-kernel timing, step
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ffn.py tests/test_gpu_fp8.py tests/test_gpu_ffn_fp8.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -3
for i in 1 2; do python scripts/kernel_bench.py --config c2 --iters 20 2>&1 | grep -E "K1|relu2|plain|K2|twin|K3|dact|sparse part"; done
python bench.py --no-e2e --no-cpu > gpurun_out/st256.json 2> gpurun_out/st256.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/st256.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','eager_ms_per_step','speedup_vs_dense')}); print(' dense', d.get('dense_twin',{}).get('ms_per_step')); print(' fp8', d.get('fp8_variant',{}).get('ms_per_step')); print(' roof', {k: d['roofline'][k] for k in ('kernel','achieved','frac')}); print(' clocks', d['clocks'])"
