set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo smoke_rc=$?
tail -5 gpurun_out/smoke1.log
timeout 900 python -m pytest tests -m gpu -q --timeout=300 -p no:cacheprovider > gpurun_out/pytest_gpu1.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/pytest_gpu1.log
timeout 900 python bench.py --steps 3 --warmup 2 --skip-cpu > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
