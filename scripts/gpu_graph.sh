timeout 900 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 -k graph 2>&1 | tail -3
timeout 600 python scripts/ab_step.py --blocks 6 --variants default,graph --dense 2>&1 | tail -1
timeout 600 python scripts/ab_step.py --blocks 6 --variants graph,default 2>&1 | tail -1
