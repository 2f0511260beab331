cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 3 --warmup 1 --skip-e2e --skip-cpu > gpurun_out/ncu_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 0 -c 1 -o gpurun_out/prof_push_r1 python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu > gpurun_out/ncu_push.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_kernel -s 6 -c 1 -o gpurun_out/prof_attn_r1 python tools/prof_attn.py 3 > gpurun_out/ncu_attn.log 2>&1; echo ncu3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_write_kernel -s 1 -c 1 -o gpurun_out/prof_write_r1 python tools/prof_attn.py 1 > gpurun_out/ncu_write.log 2>&1; echo ncu4=$?
ls gpurun_out
