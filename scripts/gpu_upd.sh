cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --kernel-name-base demangled --profile-from-start off -k "regex:k_qrcp_rr<.int.8" -s 3 -c 1 --clock-control none -o gpurun_out/qrcp_mode3 python scripts/one_factor.py cfg3 factor > gpurun_out/ncu_m3.log 2>&1
grep -v Profiling gpurun_out/ncu_m3.log | tail -3
python scripts/outliers.py cfg2 20 2>/dev/null | grep median
