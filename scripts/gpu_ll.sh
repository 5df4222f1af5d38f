cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
python scripts/one_factor.py cfg3 factor > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev/cfg3_launches.csv python scripts/one_factor.py cfg3 factor > gpurun_out/ev/ncu_list.log 2>&1
python scripts/launches.py gpurun_out/ev/cfg3_launches.csv 0 > gpurun_out/ev/cfg3_launches_summary.txt 2>&1
cat gpurun_out/ev/cfg3_launches_summary.txt
