#!/bin/bash
# fused drain + push: CTAs per SM (bitmap pass width / waves) A/B at four dirty rates
for v in 2 4 8 16 32; do
  echo "per_sm=$v"
  PL_FUSED_CTAS_PER_SM=$v timeout 200 python tools/round_latency.py 200 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items(): print(' ', k, v['keys'], 'host', v['host_us'], 'kernel', v['kernel_us'], 'wall', v['wall_us'], v['wall_us_min'])
"
done
