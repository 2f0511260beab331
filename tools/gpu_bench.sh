cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 6000 gpurun_out/bench.json; grep -v "^    " gpurun_out/bench.err | tail -20
