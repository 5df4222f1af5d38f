cd $GRAFT_REPO_ROOT
timeout 600 python scripts/alloc_trace2.py 2>&1 | tail -12
