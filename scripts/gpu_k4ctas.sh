J='import json,sys; d=json.loads(sys.stdin.read()); print({k:(v["median_ms"],v["min_ms"]) for k,v in d.items()})'
for C in 0 148 296 592 0; do
  echo "ctas $C"; S24_IDENTITY_LAYOUT=0 S24_K4_CTAS=$C timeout 600 python scripts/ab_step.py --blocks 4 --variants graph,k4_none_graph 2>&1 | tail -1 | python -c "$J"
done
