# ncu evidence of the final push kernel: launch list of the bench step, per-launch DRAM
# traffic at the bench shape, full-set capture of the bulk push
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 3 --only-step > gpurun_out/ncu_bench.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"push_batched|copy_kernel|paged_attn_mma" --csv --log-file gpurun_out/traffic_r2.csv python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-sweep --skip-c3 --skip-c2 > gpurun_out/ncu_traffic.log 2>&1; echo ncu_traffic=$?
python tools/traffic_from_csv.py gpurun_out/traffic_r2.csv gpurun_out/traffic_r2.json 80 > /dev/null; echo traffic_json=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:push_batched -s 2 -c 1 -o gpurun_out/prof_push_r2 python tools/prof_push.py 32 3 > gpurun_out/ncu_push.log 2>&1; echo ncu_push=$?
cat gpurun_out/traffic_r2.json | head -12
