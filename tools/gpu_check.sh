# smoke + GPU suite + both bench arms (the driver's round-end tiers), timed
cd $GRAFT_REPO_ROOT
t0=$(date +%s)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? $(( $(date +%s) - t0 ))s
tail -1 gpurun_out/smoke.log
t0=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -q --timeout=400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? $(( $(date +%s) - t0 ))s
tail -2 gpurun_out/pytest_gpu.log
t0=$(date +%s)
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$? $(( $(date +%s) - t0 ))s
t0=$(date +%s)
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$? $(( $(date +%s) - t0 ))s
python -c "
import json; l=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(l['value'], l['e2e']['value'], l['roofline']['frac'], l['steps'], l['warmup'])
r=json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1]); print(r['value'], r['reference_extras']['steady_round'], r['reference_extras']['scenario'])"
