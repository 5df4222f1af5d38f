cd $GRAFT_REPO_ROOT
SKB_QRCP_COOP_FIRST=1 python scripts/ab_factor.py cfg3 10
python scripts/ab_factor.py cfg3 10
SKB_QRCP_COOP_FIRST=1 SKB_QBLK_MIXED=1 python scripts/ab_factor.py cfg3 10
SKB_QRCP_COOP_FIRST=1 SKB_ENGINE_TIMING=1 python scripts/one_factor.py cfg3 factor 2>&1 | grep "engine level [123] " | tail -3
