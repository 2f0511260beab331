set -x
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_kernel -s 6 -c 1 -o gpurun_out/prof_attn_r1b python tools/prof_attn.py 3 > gpurun_out/ncu_attn_b.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_attn_b.log
