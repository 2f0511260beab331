# Round-2 validation: smoke, GPU suite, both bench arms, steady-round anatomy, ring probe, ncu.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 4000 gpurun_out/bench.json; grep -v "^    " gpurun_out/bench.err | tail -20
timeout 300 python tools/round_latency.py 20 > gpurun_out/round_latency.json 2>gpurun_out/round_latency.err; echo rl_rc=$?; cat gpurun_out/round_latency.json
for i in 1 2; do
PROBE_DUMP_S=100 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$i tools/ring_probe.py 64 2>&1 | grep -v "^\*\|OMP" | tail -2
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 3 --only-step > gpurun_out/ncu_bench.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"copy_kernel|paged_attn_mma" --csv --log-file gpurun_out/traffic_r2.csv python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-sweep --skip-c3 --skip-c2 > gpurun_out/ncu_traffic.log 2>&1; echo ncu_traffic=$?
python tools/traffic_from_csv.py gpurun_out/traffic_r2.csv gpurun_out/traffic_r2.json 80 > /dev/null; echo traffic_json=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 2 -c 1 -o gpurun_out/prof_push_r2 python tools/prof_push.py 32 3 > gpurun_out/ncu_push.log 2>&1; echo ncu_push=$?
ls gpurun_out
