cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
python scripts/one_factor.py cfg3 factor > /dev/null 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cfg3_launches_b.csv python scripts/one_factor.py cfg3 factor > /dev/null 2>&1
python scripts/launches.py gpurun_out/r02_cfg3_launches_b.csv 0 | head -12
timeout 1500 python -m pytest tests/test_gpu_large.py -q -s -x -k "cfg3 or cfg5" 2>&1 | grep -v "Warning\|fork()\|self.pid" | tail -6
timeout 900 python scripts/outliers.py cfg3 15 2>/dev/null | grep median
