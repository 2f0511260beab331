cd $GRAFT_REPO_ROOT
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_patch.py tests/test_gpu_kvstore.py tests/test_gpu_act.py -q -x -p no:cacheprovider > gpurun_out/san_mem.log 2>&1
grep -E "passed|failed|ERROR SUMMARY|^FAILED|Error|assert" gpurun_out/san_mem.log | head -30
