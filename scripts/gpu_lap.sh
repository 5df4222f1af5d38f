cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -k "laplace" 2>&1 | grep -v "Warning\|^  " | tail -25
