#!/bin/bash
# e2e in the short-repeat configuration (the one that was host-bound): three lines, with the
# slowest step's host phases and the last push's phases
mkdir -p gpurun_out/e2e_reps
timeout 300 python -m pytest tests/test_gpu_kvstore.py tests/test_gpu_staging.py -q -x 2>&1 | tail -1
for i in 1 2 3; do
  timeout 600 python bench.py --steps 10 --warmup 3 --skip-c3 --skip-sweep --skip-cpu > gpurun_out/e2e_reps/rep_$i.json 2>/dev/null
  python - "$i" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/e2e_reps/rep_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e = d["e2e"]
lp = {k: v for k, v in (e.get("last_push_phases_ms") or {}).items() if isinstance(v, float)}
print(sys.argv[1], d["value"], e["value"], e["ms_per_step"], e.get("hbm_frac"), e["host_step_ms_max"], e.get("host_step_phases_ms"), lp)
PY
done
