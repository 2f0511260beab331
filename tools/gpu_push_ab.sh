# push_batched_kernel: bench step value (FULL specialization), 4 runs, and the steady sweep
cd $GRAFT_REPO_ROOT
for m in 1 1 1 1; do
  PL_PUSH_MINB=$m timeout 600 python bench.py --steps 20 --warmup 3 --only-step > gpurun_out/pab_$m.json 2>/dev/null
  python -c "
import json; l=json.loads(open('gpurun_out/pab_$m.json').read().strip().splitlines()[-1]); print('minb $m', l['value'], l['roofline']['achieved'], l['roofline']['frac'], l['value_cold']['value'])"
done
timeout 300 python tools/round_latency.py 20 > gpurun_out/prl.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/prl.json')); print({k: (v['wall_us'], v['kernel_us']) for k, v in d.items()})"
timeout 600 python -m pytest tests/test_gpu_patch.py tests/test_gpu_fullsize.py tests/test_gpu_kvstore.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -2
