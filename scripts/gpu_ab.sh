cd $GRAFT_REPO_ROOT
timeout 900 python scripts/ab_step.py --variants graph,k4_none_graph,k4_twice_graph,act_split_bwd_graph --blocks 6 --steps 5 2>&1 | tail -2
