# compute-sanitizer memcheck over the staging-ring changes (outgrow + deferred frees,
# threaded uploads) and the patch engine
cd $GRAFT_REPO_ROOT
S=/usr/local/cuda/bin/compute-sanitizer
echo "## memcheck: test_gpu_kvstore test_gpu_patch"
timeout 1500 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kvstore.py tests/test_gpu_patch.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | head -20
echo "## memcheck: test_gpu_ipc"
timeout 900 $S --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | head -20
