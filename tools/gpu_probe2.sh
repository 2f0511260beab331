cd $GRAFT_REPO_ROOT
timeout 300 python tools/round_latency.py 30 > gpurun_out/rl_default.json 2>&1; echo rc=$?
PL_SYNC_BOOKKEEPING=1 timeout 300 python tools/round_latency.py 30 > gpurun_out/rl_sync.json 2>&1; echo rc=$?
PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 300 python tools/round_latency.py 30 > gpurun_out/rl_allfused.json 2>&1; echo rc=$?
PL_PUSH_FUSED_MAX_KEYS=0 timeout 300 python tools/round_latency.py 30 > gpurun_out/rl_nofused.json 2>&1; echo rc=$?
python - <<'PY'
import json
for f in ["rl_default","rl_sync","rl_allfused","rl_nofused"]:
    try:
        d=json.load(open(f"gpurun_out/{f}.json"))
    except Exception as e:
        print(f, "ERR", open(f"gpurun_out/{f}.json").read()[-2000:]); continue
    for k,v in d.items():
        print(f, k, "keys",v["keys"],"host",v["host_us"],"kernel",v["kernel_us"],"wall",v["wall_us"],"idle",v["host_idle_us"], v["host_phases_us"])
PY
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
