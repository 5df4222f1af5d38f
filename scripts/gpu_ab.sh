cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | grep -v "Warning\|fork()\|self.pid\|^  " | tail -3
python scripts/update_phases.py 2>&1 | head -16
python scripts/ab_factor.py cfg3 12
