# steady-round anatomy, cross-process ring control, c2 host-stall repeats
cd $GRAFT_REPO_ROOT
timeout 300 python tools/round_latency.py 30 > gpurun_out/round_latency.json 2>&1; echo rl_rc=$?
cat gpurun_out/round_latency.json | tail -60
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/ring_probe.py 64 > gpurun_out/ring_probe.txt 2>&1; echo ring_rc=$?
tail -5 gpurun_out/ring_probe.txt
PL_PATCH_SOCKET=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/ring_probe.py 64 > gpurun_out/ring_probe_socket.txt 2>&1; echo ring_rc=$?
tail -3 gpurun_out/ring_probe_socket.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 3 --only-step --skip-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
tail -c 2500 gpurun_out/bench_n2.json
for i in 1 2 3 4 5; do timeout 300 python tools/c2_probe.py > gpurun_out/c2_rep_$i.json 2>&1; echo c2_$i=$?; done
python - <<'PY'
import json
for i in range(1,6):
    try:
        d=json.loads(open(f"gpurun_out/c2_rep_{i}.json").readline())
        print(i, d["bulk"]["host_enqueue_ms"], d["bulk"]["ms"], d["switch_pause_ms"], d["decode_ms_per_step_during_bulk"])
    except Exception as e: print(i, "err", e)
PY
