cd $GRAFT_REPO_ROOT
timeout 300 python tools/round_latency.py 30 > gpurun_out/rl.json 2>/dev/null; echo rl=$?
python -c "
import json; d=json.load(open('gpurun_out/rl.json'))
for k,v in d.items(): print(k, v['keys'], 'host', v['host_us'], 'kernel', v['kernel_us'], 'wall', v['wall_us'], v['wall_us_min'])"
PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"drain_push" --csv --log-file gpurun_out/rl_launches.csv python tools/round_latency.py 4 > /dev/null 2>&1; echo ncu=$?
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/rl_launches.csv'))); h=None; v=[]
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h): v.append(round(float(dict(zip(h,r))['Metric Value'].replace(',',''))/1000,1))
print(v)
PY
timeout 900 python -m pytest tests/test_gpu_patch.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py tests/test_gpu_simulation.py -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_probe.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_probe.log
