cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"drain_push|copy_kernel|drain_compact" --csv --log-file gpurun_out/rl_launches.csv python tools/round_latency.py 5 > gpurun_out/rl_ncu.out 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:"drain_push" -s 8 -c 1 -o gpurun_out/prof_drain_push_decode python tools/round_latency.py 5 > /dev/null 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:"drain_push" -s 24 -c 1 -o gpurun_out/prof_drain_push_1pct python tools/round_latency.py 5 > /dev/null 2>&1; echo rc=$?
ls -la gpurun_out
