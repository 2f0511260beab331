set -x
cd $GRAFT_REPO_ROOT
python tools/vmm_probe.py > gpurun_out/probe.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench_rc=$?
tail -c 4000 gpurun_out/bench2.json; grep -v "^    " gpurun_out/bench2.err | tail -20
