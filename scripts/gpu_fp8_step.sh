cd $GRAFT_REPO_ROOT
timeout 900 python scripts/fp8_step.py --config c2 2>&1 | tail -40
