cd $GRAFT_REPO_ROOT
timeout 600 python scripts/update_phases.py 2>&1 | tail -30
