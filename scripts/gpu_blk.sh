cd $GRAFT_REPO_ROOT
python scripts/qrcp_bench.py
SKB_QRCP_BLK=0 python scripts/qrcp_bench.py
python scripts/qrcp_bench.py 2 1500 900 330
SKB_QRCP_BLK=0 python scripts/qrcp_bench.py 2 1500 900 330
