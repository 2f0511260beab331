cd $GRAFT_REPO_ROOT
for v in 1 2 3; do
timeout 600 python bench.py --steps 10 --warmup 3 --skip-c3 --skip-c2 --skip-sweep --skip-cpu > gpurun_out/e2e_$v.json 2>gpurun_out/e2e_$v.err; echo rc=$?
python -c "
import json; l=json.loads(open('gpurun_out/e2e_$v.json').read().strip().splitlines()[-1]); print('$v', l['value'], l['e2e']['value'], l['e2e']['ms_per_step'], l['value_cold']['value'], l['resize']['shrink_ms'])"
done
timeout 600 python tools/cold_probe.py 3 1 2>&1 | grep rep | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_kvstore.py tests/test_gpu_patch.py tests/test_gpu_fullsize.py tests/test_gpu_reference_kvstore.py -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_probe.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_probe.log
