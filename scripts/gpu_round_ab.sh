# GPU tests + interleaved A/B of the current build vs an alternative library
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -4
timeout 600 python scripts/ab_step.py --blocks 6 --dense 2>&1 | tail -2
for i in 1 2; do
  for L in "" ${ALT_LIB}; do
    echo "== lib [$L]"; S24_LIB=$L timeout 300 python scripts/ab_step.py --blocks 4 --variants default 2>&1 | tail -1
  done
done
timeout 300 python scripts/kernel_bench.py 2>&1 | grep "K4\|K7\|K6"
