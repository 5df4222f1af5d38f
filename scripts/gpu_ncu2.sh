cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --profile-from-start off -k regex:k_qrcp2 -s 11 -c 1 --clock-control none -o gpurun_out/qrcp2_mode2 python scripts/one_factor.py cfg3 factor > gpurun_out/ncu2.log 2>&1
grep -v "Profiling" gpurun_out/ncu2.log | tail -3
