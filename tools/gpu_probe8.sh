cd $GRAFT_REPO_ROOT
PROBE_DUMP_S=100 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/ring_probe.py 64 > gpurun_out/ring_probe.txt 2>&1; echo ring_rc=$?
grep -v "^\*\|OMP" gpurun_out/ring_probe.txt | tail -6
timeout 600 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_dist_llama.py tests/test_gpu_act.py tests/test_gpu_model8b.py -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 3 --only-step --skip-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
python -c "
import json; l=json.loads(open('gpurun_out/bench_n2.json').read().strip().splitlines()[-1]); print(l['value'], l['roofline'])"
