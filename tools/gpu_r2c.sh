# Round-2 evidence run (after the pause / cold-round work): smoke, GPU suite, both bench
# arms, steady-round anatomy, 4 repeated bench runs, configs[3] x3, 2-rank ring on one GPU
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 2500 gpurun_out/bench.json; grep -v "^    " gpurun_out/bench.err | tail -5
timeout 300 python tools/round_latency.py 30 > gpurun_out/round_latency.json 2>/dev/null; echo rl_rc=$?
for i in 1 2 3 4; do
  timeout 600 python bench.py --steps 10 --warmup 3 --skip-c3 --skip-sweep --skip-cpu --skip-e2e > gpurun_out/rep_$i.json 2>/dev/null; echo rep_$i=$?
done
for i in 1 2 3; do
  timeout 400 python tools/c4_live.py > gpurun_out/c4_$i.json 2>gpurun_out/c4_$i.err; echo c4_$i=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 3 --only-step > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
tail -c 1500 gpurun_out/bench_n2.json
for i in 1 2; do
PROBE_DUMP_S=100 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$i tools/ring_probe.py 64 2>&1 | grep -v "^\*\|OMP" | tail -2
done
PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 600 ncu --set full --clock-control none --import-source on -k regex:drain_push -s 4 -c 1 -o gpurun_out/prof_steady_decode_r2 python tools/round_latency.py 4 > gpurun_out/ncu_steady.log 2>&1; echo ncu_steady=$?
