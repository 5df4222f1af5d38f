cd $GRAFT_REPO_ROOT
python scripts/timeline.py cfg3 factor gpurun_out/tl_f.json -v > gpurun_out/tl_cfg3_factor.txt 2>&1
rm -f gpurun_out/tl_f.json
python scripts/timeline.py cfg2 update gpurun_out/tl_upd.json -v > gpurun_out/tl_cfg2_update.txt 2>&1
rm -f gpurun_out/tl_upd.json
python scripts/update_phases.py > gpurun_out/update_phases.txt 2>&1
head -8 gpurun_out/tl_cfg3_factor.txt gpurun_out/tl_cfg2_update.txt
