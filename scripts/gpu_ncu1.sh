cd $GRAFT_REPO_ROOT
python scripts/one_factor.py cfg3 factor > /dev/null 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_cfg3_launches.csv python scripts/one_factor.py cfg3 factor > gpurun_out/ncu1.log 2>&1
python scripts/launches.py gpurun_out/r02_cfg3_launches.csv 25 | head -60
