cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_active.avg,launch__grid_size,smsp__cycles_active.max
for cps in 2 1 8; do
PL_FUSED_CTAS_PER_SM=$cps PL_PUSH_FUSED_MAX_KEYS=100000000 ncu --metrics $M --clock-control none -k regex:"drain_push" -c 30 --csv --log-file gpurun_out/fp_$cps.csv python tools/round_latency.py 5 > /dev/null 2>&1; echo rc=$?
done
PL_PUSH_FUSED_MAX_KEYS=100000000 ncu --metrics $M --cache-control none --clock-control none -k regex:"drain_push" -c 30 --csv --log-file gpurun_out/fp_nocache.csv python tools/round_latency.py 5 > /dev/null 2>&1; echo rc=$?
