cd $GRAFT_REPO_ROOT
for v in 1 0; do
echo "BLK=$v"
SKB_QRCP_BLK=$v SKB_ENGINE_TIMING=1 python scripts/one_factor.py cfg3 factor 2>&1 | grep "level [123] " | tail -6
done
