# Round-2 final evidence: smoke, GPU suite, both bench arms (full line), repeats, configs[3]
# runs, steady-round anatomy, 2-rank ring, ncu launch list / traffic / full captures
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "
import json; l=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(l['value'], l['e2e']['value'], l['roofline']['frac'], json.dumps(l['tail'])[:1600])"
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --steps 10 --warmup 3 --skip-c3 --skip-sweep --skip-cpu > gpurun_out/rep_$i.json 2>/dev/null; echo rep_$i=$?
done
for i in 1 2 3; do
  timeout 400 python tools/c4_live.py > gpurun_out/c4_$i.json 2>gpurun_out/c4_$i.err; echo c4_$i=$?
done
timeout 300 python tools/round_latency.py 30 > gpurun_out/round_latency.json 2>/dev/null; echo rl_rc=$?
timeout 300 python tools/e2e_timeline.py 20 > gpurun_out/e2e_timeline.txt 2>&1; echo tl_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 3 --only-step > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 3 --only-step > gpurun_out/ncu_bench.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"push_batched|copy_kernel|paged_attn_mma" --csv --log-file gpurun_out/traffic_r2.csv python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-sweep --skip-c3 --skip-c2 > gpurun_out/ncu_traffic.log 2>&1; echo ncu_traffic=$?
python tools/traffic_from_csv.py gpurun_out/traffic_r2.csv gpurun_out/traffic_r2.json 80 > /dev/null; echo traffic_json=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:push_batched -s 2 -c 1 -o gpurun_out/prof_push_r2 python tools/prof_push.py 32 3 > gpurun_out/ncu_push.log 2>&1; echo ncu_push=$?
PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:drain_push -s 4 -c 1 -o gpurun_out/prof_steady_decode_r2 python tools/round_latency.py 4 > gpurun_out/ncu_steady.log 2>&1; echo ncu_steady=$?
PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:drain_push -s 20 -c 1 -o gpurun_out/prof_steady_r2 python tools/round_latency.py 4 > gpurun_out/ncu_steady1.log 2>&1; echo ncu_steady1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_write -s 3 -c 1 -o gpurun_out/prof_k1_r2 python tools/e2e_timeline.py 2 > gpurun_out/ncu_k1.log 2>&1; echo ncu_k1=$?
ls gpurun_out
