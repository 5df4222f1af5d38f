cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k getrf 2>&1 | tail -2
LU_BREAKDOWN=1 timeout 300 python scripts/lu_bench.py 849 2532 2>&1 | tail -4
