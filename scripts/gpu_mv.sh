cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "move" 2>&1 | tail -15
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | grep -v "Warning\|fork()\|self.pid\|^  " | tail -5
python scripts/ab_factor.py cfg3 12
python scripts/ab_factor.py cfg2 12
python scripts/upd_bench.py
python scripts/solve_bench.py 2>&1 | tail -3
