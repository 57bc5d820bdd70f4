timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -3
timeout 600 python scripts/ab_step.py --blocks 4 --variants graph,default 2>&1 | tail -1 | cut -c1-200
S24_PAIRED_DENSE=0 timeout 600 python scripts/ab_step.py --blocks 4 --variants graph,default 2>&1 | tail -1 | cut -c1-200
timeout 600 python scripts/ab_step.py --blocks 4 --variants graph,default 2>&1 | tail -1 | cut -c1-200
