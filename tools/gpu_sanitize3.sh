# compute-sanitizer memcheck over the attention, cross-process and 8B-shape suites
cd $GRAFT_REPO_ROOT
S=/usr/local/cuda/bin/compute-sanitizer
for t in tests/test_gpu_attention.py tests/test_gpu_ipc.py tests/test_gpu_model8b.py tests/test_gpu_fullsize.py; do
  echo "## memcheck: $t"
  timeout 1500 $S --tool memcheck --target-processes all python -m pytest $t -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | tail -4
done
