# batched-resolve push A/B (round latency, sweep, headline step), random-copy floor,
# kernel-only durations under ncu, model8b live switch
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rcp tools/rand_copy_probe.cu -lcuda && timeout 120 /tmp/rcp 4 128 2621 13107 65536 > gpurun_out/rcp.txt 2>&1; echo rcp=$?; cat gpurun_out/rcp.txt
for b in 1 0; do
  PL_PUSH_BATCHED=$b timeout 300 python tools/round_latency.py 30 > gpurun_out/rl_b$b.json 2>/dev/null; echo rl_b$b=$?
  PL_PUSH_BATCHED=$b timeout 300 python bench.py --steps 10 --warmup 3 --only-step --skip-e2e > gpurun_out/step_b$b.json 2>/dev/null; echo step_b$b=$?
done
python - <<'PY'
import json
for b in (1, 0):
    d=json.load(open(f"gpurun_out/rl_b{b}.json"))
    for k,v in d.items():
        print("batched",b, k, "keys",v["keys"],"host",v["host_us"],"kernel",v["kernel_us"],"wall",v["wall_us"],"idle",v["host_idle_us"])
    l=json.loads(open(f"gpurun_out/step_b{b}.json").read().strip().splitlines()[-1])
    print("batched", b, "value", l["value"], l["roofline"])
PY
for b in 1 0; do
PL_PUSH_BATCHED=$b timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"drain_push|copy_kernel|drain_compact|push_batched" --csv --log-file gpurun_out/rl_launches_b$b.csv python tools/round_latency.py 4 > /dev/null 2>&1; echo ncu_b$b=$?
done
timeout 600 python -m pytest tests/test_gpu_model8b.py tests/test_gpu_patch.py tests/test_gpu_ipc.py -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_probe.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_probe.log
timeout 600 python tools/c2_model_probe.py > gpurun_out/c2_model.json 2>gpurun_out/c2_model.err; echo c2m=$?
python -c "
import json; d=json.load(open('gpurun_out/c2_model.json')); print({k:d[k] for k in d if k not in ('lag_polls',)})"
