cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_act.py tests/test_gpu_ipc.py tests/test_gpu_dist_llama.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 10 --warmup 3 --only-step > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
python -c "
import json; l=json.loads(open('gpurun_out/bench_n2.json').read().strip().splitlines()[-1]); print(l['value'], l['roofline']['frac'], l['value_cold'])"
PROBE_DUMP_S=100 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/ring_probe.py 64 2>&1 | grep -v "^\*\|OMP" | tail -2
timeout 400 python tools/c4_live.py > gpurun_out/c4_x.json 2>gpurun_out/c4_x.err; echo c4=$?
python -c "
import json; d=json.load(open('gpurun_out/c4_live.json')); print(d['steps']['pause_ms'])"
