cd $GRAFT_REPO_ROOT
PL_TRACE_PUSH=1 timeout 600 python tools/cold_probe.py 3 1 > gpurun_out/cold_w1.txt 2>&1; echo rc=$?; grep -v "^\[pl\] reclaim\|ensure:" gpurun_out/cold_w1.txt | tail -12
PL_PUSH_NO_CHUNK=1 PL_TRACE_PUSH=1 timeout 600 python tools/cold_probe.py 2 1 > gpurun_out/cold_nochunk.txt 2>&1; echo rc=$?; grep -v "^\[pl\] reclaim\|ensure:" gpurun_out/cold_nochunk.txt | tail -8
timeout 900 python -m pytest tests/test_gpu_kvstore.py tests/test_gpu_patch.py tests/test_gpu_ipc.py tests/test_gpu_simulation.py tests/test_gpu_fullsize.py -q -x --timeout=400 -p no:cacheprovider > gpurun_out/pytest_probe.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_probe.log
