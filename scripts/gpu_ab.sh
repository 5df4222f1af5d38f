cd $GRAFT_REPO_ROOT
SKB_ENGINE_TIMING=1 python scripts/upd3_outliers.py nosolve > gpurun_out/u3.txt 2>&1
grep "^move" gpurun_out/u3.txt
