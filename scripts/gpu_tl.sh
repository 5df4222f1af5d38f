cd $GRAFT_REPO_ROOT
python scripts/timeline.py cfg2 update gpurun_out/tl_upd.json -v > gpurun_out/tl_cfg2_update.txt 2>&1
head -8 gpurun_out/tl_cfg2_update.txt
rm -f gpurun_out/tl_upd.json
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | grep -v "Warning\|fork()\|self.pid\|^  " | tail -4
