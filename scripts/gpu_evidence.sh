# Round-2 evidence run: tests, bench (driver settings), reference arm, ncu launch list + captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev/smi.txt
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | grep -v "Warning\|fork()\|self.pid\|^  " | tail -6 > gpurun_out/ev/gpu_tests.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
python scripts/one_factor.py cfg3 factor > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev/r02_cfg3_launches.csv python scripts/one_factor.py cfg3 factor > gpurun_out/ev/ncu_list.log 2>&1
python scripts/launches.py gpurun_out/ev/r02_cfg3_launches.csv 0 > gpurun_out/ev/r02_cfg3_launches_summary.txt 2>&1
python scripts/ncu_traffic.py gpurun_out/ev/r02_cfg3_launches.csv gpurun_out/ev/r02_cfg3_traffic.json > gpurun_out/ev/traffic.txt 2>&1
# full captures of the top kernels (one launch each)
for spec in "k_assemble_stack:3" "k_qrcp2:11" "k_qrcp_blk:0" "k_qrcp_rr:5" "k_gemm_grouped:40" "k_getf2_cl:10" "k_geqrf_cl:4" "k_geqrf_box:4" "k_gather_rows:20"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --profile-from-start off -k regex:$k -s $s -c 1 --clock-control none -o /tmp/full_$k python scripts/one_factor.py cfg3 factor > gpurun_out/ev/ncu_$k.log 2>&1
done
# summaries only travel back (the .ncu-rep files exceed the 64 MiB return limit)
python scripts/ncu_summary.py /tmp/full_*.ncu-rep > gpurun_out/ev/r02_ncu_full_captures.txt 2>&1
rm -f gpurun_out/ev/ncu_k_*.log
python scripts/one_factor.py cfg2 update > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/r02_cfg2_update_launches.csv python scripts/one_factor.py cfg2 update > gpurun_out/ev/ncu_upd.log 2>&1
python scripts/launches.py gpurun_out/ev/r02_cfg2_update_launches.csv 0 > gpurun_out/ev/r02_cfg2_update_launches_summary.txt 2>&1
python scripts/qrcp_bench.py > gpurun_out/ev/qrcp_bench.txt 2>&1
SKB_QRCP_BLK=0 python scripts/qrcp_bench.py >> gpurun_out/ev/qrcp_bench.txt 2>&1
ls -la gpurun_out/ev
