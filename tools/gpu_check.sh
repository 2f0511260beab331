# smoke + GPU suite + bench (the driver's round-end tiers)
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "
import json; l=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(l['value'], l['e2e'], l['roofline']['frac'], json.dumps(l['tail'])[:900])"
