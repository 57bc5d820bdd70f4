J='import json,sys; d=json.loads(sys.stdin.read()); print({k:(v["median_ms"],v["min_ms"]) for k,v in d.items()})'
for L in "" paper_2503_16672_b200/_exp/libs24_k4x5.so; do
echo "== [$L]"
S24_LIB=$L timeout 600 python scripts/ab_step.py --blocks 5 --variants graph,act_split_bwd_graph,k4_none_graph 2>&1 | tail -1 | python -c "$J"
S24_LIB=$L timeout 600 python scripts/ab_step.py --blocks 5 --variants act_split_bwd_graph,graph,k4_none_graph 2>&1 | tail -1 | python -c "$J"
done
