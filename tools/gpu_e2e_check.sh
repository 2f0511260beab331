#!/bin/bash
# e2e host-stall check: the staging-ring test, the stall probe, three full bench lines
set -x
mkdir -p gpurun_out/e2e_check
timeout 300 python -m pytest tests/test_gpu_kvstore.py -q -x -k "upload_ring or replays_reference" 2>&1 | tail -3
timeout 600 python tools/e2e_stall_probe.py --steps 20 --reps 3 > gpurun_out/e2e_check/probe.log 2>&1
tail -12 gpurun_out/e2e_check/probe.log | cut -c1-200
for i in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/e2e_check/bench_$i.json 2> gpurun_out/e2e_check/bench_$i.err
  python - "$i" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/e2e_check/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(sys.argv[1], d["value"], e["value"], e["ms_per_step"], e["host_step_ms_max"], e.get("host_step_phases_ms"), e.get("staging"))
PY
done
