# K1 write order A/B (PL_K1_LAYER_MAJOR): e2e timeline K1 time, e2e bench, byte-exact suites
cd $GRAFT_REPO_ROOT
for m in 0 1 0 1; do
  PL_K1_LAYER_MAJOR=$m timeout 300 python tools/e2e_timeline.py 20 2>&1 | grep -E "kv_write|wall" | head -2 | sed "s/^/lm=$m /"
done
for m in 0 1; do
  PL_K1_LAYER_MAJOR=$m timeout 600 python bench.py --steps 10 --warmup 3 --skip-c3 --skip-c2 --skip-sweep --skip-cpu > gpurun_out/k1_$m.json 2>/dev/null
  python -c "
import json; l=json.loads(open('gpurun_out/k1_$m.json').read().strip().splitlines()[-1]); print('lm $m', l['value'], l['e2e']['value'], l['e2e']['ms_per_step'])"
done
PL_K1_LAYER_MAJOR=1 timeout 900 python -m pytest tests/test_gpu_kvstore.py tests/test_gpu_fullsize.py tests/test_gpu_patch.py tests/test_gpu_reference_kvstore.py tests/test_gpu_llama.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -2
