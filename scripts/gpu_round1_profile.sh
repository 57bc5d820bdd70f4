set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo rc=$?
tail -c 3000 gpurun_out/bench_r1.json
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/plain_small.json 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_launch.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:GemmCfgILb1E.*EpiStoreIfE' -s 4 -c 1 -o gpurun_out/prof_dw_sparse python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_dw.log 2>&1; echo rc=$?
tail -5 gpurun_out/ncu_dw.log
