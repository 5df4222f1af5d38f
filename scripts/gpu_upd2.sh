cd $GRAFT_REPO_ROOT
timeout 600 python scripts/inc_check.py 2>&1 | tail -12
