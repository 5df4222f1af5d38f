cd $GRAFT_REPO_ROOT
SKB_ENGINE_TIMING=1 python scripts/timeline.py cfg3 factor gpurun_out/tl_cfg3.json -v > gpurun_out/tl_cfg3.txt 2> gpurun_out/tl_cfg3.err
head -12 gpurun_out/tl_cfg3.txt; grep "engine level" gpurun_out/tl_cfg3.err | tail -12
python scripts/timeline.py cfg2 update gpurun_out/tl_cfg2u.json -v > gpurun_out/tl_cfg2u.txt 2>&1; head -12 gpurun_out/tl_cfg2u.txt
rm -f gpurun_out/tl_cfg3.json gpurun_out/tl_cfg2u.json
