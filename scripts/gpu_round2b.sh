cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -s -m gpu -k "interior or unphased or tie_rich or replay" 2>&1 | grep -v "^  \|Warning" | tail -30
