cd $GRAFT_REPO_ROOT
timeout 300 python tools/round_latency.py 30 > gpurun_out/rl_default.json 2>&1; echo rc=$?
python - <<'PY'
import json
d=json.load(open("gpurun_out/rl_default.json"))
for k,v in d.items():
    print(k, "keys",v["keys"],"host",v["host_us"],"kernel",v["kernel_us"],"wall",v["wall_us"],"idle",v["host_idle_us"], v["host_phases_us"])
PY
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/ring_probe.py 64 > gpurun_out/ring_probe.txt 2>&1; echo ring_rc=$?
grep -v "^\*\|OMP" gpurun_out/ring_probe.txt | tail -6
timeout 900 python -m pytest tests/test_gpu_patch.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
