#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense"
timeout 300 $B > gpurun_out/prof_plain.json 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:GemmCfgILb1ELb0ELb1E.*EpiStoreIfLb0E" -s 6 -c 1 -o gpurun_out/prof_spmm_pair $B > gpurun_out/ncu_spmm_pair.log 2>&1; echo pair rc=$?
python scripts/ncu_summary.py gpurun_out/prof_spmm_pair.ncu-rep > gpurun_out/ncu_spmm_pair_v4.txt 2>&1
tail -3 gpurun_out/ncu_spmm_pair.log
