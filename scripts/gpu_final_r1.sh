# bench (default) + reference arm + launch list + full captures of the top kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_r1_final.json 2>gpurun_out/bench_r1_final.err; echo bench rc=$?
tail -c 2500 gpurun_out/bench_r1_final.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?; tail -c 600 gpurun_out/bench_ref.json
bash scripts/gpu_profiles.sh
