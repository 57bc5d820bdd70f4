cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck.log 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/memcheck.log
grep -c "Invalid\|ERROR SUMMARY" gpurun_out/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_fp8.py -q -x -k "quant_rows_bitwise or quant_cols or meta or spmm_f8" > gpurun_out/racecheck.log 2>&1; echo racecheck rc=$?
tail -5 gpurun_out/racecheck.log
