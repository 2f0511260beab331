cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_patch.py tests/test_gpu_ipc.py tests/test_gpu_fullsize.py tests/test_gpu_simulation.py tests/test_gpu_reference_migrator.py tests/test_gpu_llama.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/round_latency.py 30 > gpurun_out/rl.json 2>/dev/null; echo rl=$?
python -c "
import json; d=json.load(open('gpurun_out/rl.json'))
for k,v in d.items(): print(k, v['keys'], 'host', v['host_us'], 'kernel', v['kernel_us'], 'wall', v['wall_us'], v['wall_us_min'])"
