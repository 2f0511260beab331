# ncu evidence for the bench: launch list, per-launch DRAM traffic, full-set captures.
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 3 --warmup 3 --only-step > gpurun_out/ncu_bench.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"copy_kernel|paged_attn_mma" --csv --log-file gpurun_out/traffic_r1.csv python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-sweep --skip-c3 --skip-c2 > gpurun_out/ncu_traffic.log 2>&1; echo ncu_traffic=$?
python tools/traffic_from_csv.py gpurun_out/traffic_r1.csv gpurun_out/traffic_r1.json 80 > /dev/null; echo traffic_json=$?
