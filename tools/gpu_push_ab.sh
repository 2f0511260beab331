# push lane order by density: bench step + steady sweep + parity suites
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_patch.py tests/test_gpu_fullsize.py tests/test_gpu_ipc.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -1
for m in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --only-step > gpurun_out/pab_$m.json 2>/dev/null
  python -c "
import json; l=json.loads(open('gpurun_out/pab_$m.json').read().strip().splitlines()[-1]); print('run $m', l['value'], l['roofline']['achieved'], l['roofline']['frac'], l['value_cold']['value'])"
done
timeout 300 python tools/round_latency.py 20 > gpurun_out/prl.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/prl.json')); print({k: (v['wall_us'], v['kernel_us']) for k, v in d.items()})"
