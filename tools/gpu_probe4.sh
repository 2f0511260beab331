cd $GRAFT_REPO_ROOT
for v in default allfused nofused; do
  case $v in allfused) export PL_PUSH_FUSED_MAX_KEYS=100000000;; nofused) export PL_PUSH_FUSED_MAX_KEYS=0;; *) unset PL_PUSH_FUSED_MAX_KEYS;; esac
  timeout 300 python tools/round_latency.py 30 > gpurun_out/rl_$v.json 2>&1; echo rc=$?
done
unset PL_PUSH_FUSED_MAX_KEYS
python - <<'PY'
import json
for f in ["rl_default","rl_allfused","rl_nofused"]:
    try: d=json.load(open(f"gpurun_out/{f}.json"))
    except Exception as e: print(f, "ERR", open(f"gpurun_out/{f}.json").read()[-2000:]); continue
    for k,v in d.items():
        print(f, k, "keys",v["keys"],"host",v["host_us"],"kernel",v["kernel_us"],"wall",v["wall_us"],"idle",v["host_idle_us"], v["host_phases_us"])
PY
PL_PUSH_FUSED_MAX_KEYS=100000000 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"drain_push|copy_kernel|drain_compact" --csv --log-file gpurun_out/rl_launches.csv python tools/round_latency.py 5 > gpurun_out/rl_ncu.out 2>&1; echo rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
