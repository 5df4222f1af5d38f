cd $GRAFT_REPO_ROOT
export RACE_MAXLEV=2
(SKB_ENGINE_LEAD=-1 SKB_ENGINE_SNAP=1 timeout 600 python scripts/race_hunt.py 60 6) > gpurun_out/race_lead.json 2> gpurun_out/race_lead.err
(timeout 600 python scripts/race_hunt.py 60 6) > gpurun_out/race_default.json 2> gpurun_out/race_default.err
tail -c 1500 gpurun_out/race_*.json
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
