cd $GRAFT_REPO_ROOT
python scripts/upd_bench.py
SKB_QRCP_CMIN=8 python scripts/upd_bench.py
SKB_QRCP_CMIN=16 python scripts/upd_bench.py
SKB_QRCP_CMIN=8 python scripts/ab_factor.py cfg2 12
SKB_QRCP_CMIN=16 python scripts/ab_factor.py cfg2 12
SKB_QRCP_CMIN=8 python scripts/ab_factor.py cfg3 12
