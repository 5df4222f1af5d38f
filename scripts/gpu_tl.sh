cd $GRAFT_REPO_ROOT
SKB_HOST_PROF=trace python scripts/timeline.py cfg2 update gpurun_out/tl_cfg2u.json -v > gpurun_out/tl_cfg2u.txt 2>&1; head -4 gpurun_out/tl_cfg2u.txt
rm -f gpurun_out/tl_cfg2u.json
