timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -1
timeout 300 python scripts/kernel_bench.py 2>&1 | grep "sparse" | cut -c1-100
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:GemmCfgILb1ELb0ELb1E.*EpiStoreIfE" -s 6 -c 1 -o gpurun_out/prof_spmm_pair $B > gpurun_out/ncu_spmm_pair.log 2>&1; echo pair rc=$?
