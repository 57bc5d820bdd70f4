cd $GRAFT_REPO_ROOT
timeout 900 python scripts/kernel_bench.py --config c2 --iters 10 2>&1 | tail -30
