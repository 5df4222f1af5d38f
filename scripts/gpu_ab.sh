cd $GRAFT_REPO_ROOT
python scripts/ab_factor.py cfg3 10
SKB_QRCP_SMEM_FIRST=1 python scripts/ab_factor.py cfg3 10
python scripts/ab_factor.py cfg2 10
SKB_QRCP_SMEM_FIRST=1 python scripts/ab_factor.py cfg2 10
