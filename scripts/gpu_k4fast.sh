J='import json,sys; d=json.loads(sys.stdin.read()); print({k:(v["median_ms"],v["min_ms"]) for k,v in d.items()})'
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 -k "feature_split or split_weight" 2>&1 | tail -1
timeout 300 python scripts/kernel_bench.py 2>&1 | grep "K4"
timeout 600 python scripts/ab_step.py --blocks 5 --variants graph,k4_none_graph 2>&1 | tail -1 | python -c "$J"
