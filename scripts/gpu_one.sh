cd $GRAFT_REPO_ROOT
python scripts/det_check2.py mini_holes 2>&1 | grep -v "Exception ignored\|Traceback\|File \|AttributeError" | tail -20
