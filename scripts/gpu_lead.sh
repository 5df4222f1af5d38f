cd $GRAFT_REPO_ROOT
SKB_ENGINE_LEAD=1 python scripts/stall_hunt.py 150 2>&1 | head -4
SKB_ENGINE_LEAD=1 SKB_PREWARM_KB_PER_DOF=0 python scripts/stall_hunt.py 150 2>&1 | head -4
