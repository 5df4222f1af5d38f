cd $GRAFT_REPO_ROOT
timeout 2000 python -m pytest tests/test_gpu_large.py -q -s 2>&1 | grep -v "Warning\|fork()\|self.pid" | tail -25
