cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ffn.py -q --timeout 500 -k "wgrad or graph" 2>&1 | tail -3
timeout 900 python scripts/ab_step.py --variants graph,wgrad_overlap_graph --blocks 8 --steps 5 2>&1 | tail -3
