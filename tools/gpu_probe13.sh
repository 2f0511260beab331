cd $GRAFT_REPO_ROOT
PL_TRACE_PUSH=1 timeout 600 python tools/cold_probe.py 3 1 > gpurun_out/cold_w1.txt 2>&1; echo rc=$?; grep -v "^\[pl\] reclaim\|ensure:" gpurun_out/cold_w1.txt | tail -12
PL_TRACE_PUSH=1 timeout 600 python tools/cold_probe.py 2 0 > gpurun_out/cold_w0.txt 2>&1; echo rc=$?; grep -v "^\[pl\] reclaim\|ensure:" gpurun_out/cold_w0.txt | tail -8
PL_PUSH_NO_CHUNK=1 PL_TRACE_PUSH=1 timeout 600 python tools/cold_probe.py 2 1 > gpurun_out/cold_nochunk.txt 2>&1; echo rc=$?; grep -v "^\[pl\] reclaim\|ensure:" gpurun_out/cold_nochunk.txt | tail -8
