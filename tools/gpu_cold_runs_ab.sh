#!/bin/bash
# cold bulk round (value_cold): fixed 1/8 runs vs doubling runs (PL_PUSH_RUN_GROW), alternated
for rep in 1 2; do
  for g in 0 1; do
    echo "grow=$g rep=$rep"
    PL_PUSH_RUN_GROW=$g timeout 300 python tools/cold_probe.py 6 2>/dev/null | python -c "
import json,sys
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
for r in rows[1:]: print('  gbs', r['gbs'], 'wall', r['wall_ms'], 'copy', r['copy_device_ms'], 'launches', r['copy_launches'], 'pre', r['phases_ms'].get('k3_enqueue'), 'reserve', r['phases_ms'].get('reserve'))
"
  done
done
