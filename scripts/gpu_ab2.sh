timeout 900 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 2>&1 | tail -2
S24_SIDE_GATHERS=0 timeout 900 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 2>&1 | tail -2
timeout 600 python scripts/ab_step.py --blocks 6 --variants default,main_gathers 2>&1 | tail -1
timeout 600 python scripts/ab_step.py --blocks 6 --variants main_gathers,default 2>&1 | tail -1
