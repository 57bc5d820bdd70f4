#!/bin/bash
# end-of-round refresh: full default bench line, then the launch list and ncu captures
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?
tail -c 400 gpurun_out/bench_c2.err
bash scripts/gpu_profiles.sh
for r in spmm_fwdout spmm_pair k1 k3 k4; do
  [ -f gpurun_out/prof_$r.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/ncu_${r}_v4.txt 2>&1
done
ls gpurun_out/
