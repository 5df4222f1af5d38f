cd $GRAFT_REPO_ROOT
python scripts/upd_bench.py
python scripts/ab_factor.py cfg3 16
