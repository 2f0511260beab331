# fused drain+push with batched resolve + host trims: round latency, ncu kernel times, patch tests
cd $GRAFT_REPO_ROOT
timeout 300 python tools/round_latency.py 30 > gpurun_out/rl12.json 2>/dev/null; echo rl=$?
PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 300 python tools/round_latency.py 30 > gpurun_out/rl12_allfused.json 2>/dev/null; echo rl=$?
python - <<'PY'
import json
for f in ("rl12", "rl12_allfused"):
    d=json.load(open(f"gpurun_out/{f}.json"))
    for k,v in d.items():
        print(f, k, "keys",v["keys"],"host",v["host_us"],"kernel",v["kernel_us"],"wall",v["wall_us"],"min",v["wall_us_min"],"idle",v["host_idle_us"], v["host_phases_us"])
PY
PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"drain_push" --csv --log-file gpurun_out/rl12_launches.csv python tools/round_latency.py 4 > /dev/null 2>&1; echo ncu=$?
timeout 900 python -m pytest tests/test_gpu_patch.py tests/test_gpu_ipc.py tests/test_gpu_simulation.py tests/test_gpu_fullsize.py -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_probe.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_probe.log
