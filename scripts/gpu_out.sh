cd $GRAFT_REPO_ROOT
for lead in -1 1 0; do
SKB_ENGINE_LEAD=$lead timeout 900 python scripts/outliers.py cfg3 40 2>/dev/null | grep median | sed "s/^/lead $lead: /"
done
