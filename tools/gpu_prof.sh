set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --id=0 --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > gpurun_out/clocks_test.csv 2> gpurun_out/clocks_test.err &
CP=$!; sleep 2; kill $CP
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --skip-e2e --skip-cpu > gpurun_out/ncu_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 2 -c 1 -o gpurun_out/prof_push_r1 python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu > gpurun_out/ncu_push.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_attn_kernel -s 4 -c 1 -o gpurun_out/prof_attn_r1 python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu > gpurun_out/ncu_attn.log 2>&1; echo ncu3=$?
ls -la gpurun_out
