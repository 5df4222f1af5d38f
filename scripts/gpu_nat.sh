cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | grep -v "Warning\|fork()\|self.pid\|^  " | tail -15
python scripts/update_phases.py 2>&1 | tail -30
python scripts/ab_factor.py cfg2 12
python scripts/ab_factor.py cfg3 12
