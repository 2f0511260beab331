cd $GRAFT_REPO_ROOT
PL_TRACE_PUSH=1 timeout 600 python tools/cold_probe.py 4 1 2>&1 | grep -E "^\{|chunked" | cut -c1-260
timeout 600 python -m pytest tests/test_gpu_patch.py tests/test_gpu_fullsize.py -q -x --timeout=400 -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --only-step > gpurun_out/cold_$i.json 2>/dev/null
python -c "
import json; l=json.loads(open('gpurun_out/cold_$i.json').read().strip().splitlines()[-1]); print(l['value'], l['value_cold'])"
done
