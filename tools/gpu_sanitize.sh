# compute-sanitizer passes over the round-2 kernels (push_batched, drain_push, K1, verify,
# exact mode, K7 rings); each pass bounded by timeout
cd $GRAFT_REPO_ROOT
S=/usr/local/cuda/bin/compute-sanitizer
echo "## memcheck: test_gpu_patch test_gpu_kvstore test_gpu_act"
timeout 1200 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_patch.py tests/test_gpu_kvstore.py tests/test_gpu_act.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | head -20
echo "## memcheck: test_gpu_llama (exact mode) test_gpu_model8b -k small"
timeout 1200 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_llama.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid" | head -20
echo "## racecheck: test_gpu_patch -k 'push or fused or steady or drain'"
timeout 1200 $S --tool racecheck python -m pytest tests/test_gpu_patch.py -q -x -p no:cacheprovider -k "push or fused or steady or drain" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY" | head -10
echo "## synccheck: test_gpu_patch -k 'push or fused or steady or drain'"
timeout 1200 $S --tool synccheck python -m pytest tests/test_gpu_patch.py -q -x -p no:cacheprovider -k "push or fused or steady or drain" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | head -10
