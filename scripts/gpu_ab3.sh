S24_ROWMAP=0 timeout 900 python -m pytest tests/test_gpu_ffn.py -x -q --timeout 300 2>&1 | tail -1
timeout 600 python scripts/ab_step.py --blocks 6 --variants default,no_rowmap,main_gathers 2>&1 | tail -1
timeout 600 python scripts/ab_step.py --blocks 6 --variants no_rowmap,main_gathers,default 2>&1 | tail -1
timeout 600 python scripts/ab_step.py --blocks 6 --variants main_gathers,default,no_rowmap 2>&1 | tail -1
