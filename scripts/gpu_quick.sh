timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -1
timeout 300 python scripts/kernel_bench.py 2>&1 | grep -v "K7\|K4\|K6" | cut -c1-100
timeout 300 python scripts/ab_step.py --blocks 3 --variants graph,default 2>&1 | tail -1 | cut -c1-200
