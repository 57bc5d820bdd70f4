J='import json,sys; d=json.loads(sys.stdin.read()); print({k:(v["median_ms"],v["min_ms"]) for k,v in d.items()})'
timeout 600 python scripts/ab_step.py --blocks 5 --variants graph,fused_fw_graph,k4_none_graph 2>&1 | tail -1 | python -c "$J"
timeout 600 python scripts/ab_step.py --blocks 5 --variants fused_fw_graph,k4_none_graph,graph 2>&1 | tail -1 | python -c "$J"
