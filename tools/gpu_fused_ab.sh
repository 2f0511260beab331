# fused drain+push variants (PL_FUSED_VARIANT) at the decode pattern and 1/5/25 % dirty,
# every round forced through the fused kernel; kernel durations from the ncu launch list
cd $GRAFT_REPO_ROOT
for v in 0 1 2 3; do
  PL_FUSED_VARIANT=$v PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 300 python tools/round_latency.py 20 > gpurun_out/rlv$v.json 2>/dev/null
  PL_FUSED_VARIANT=$v PL_PUSH_FUSED_MAX_KEYS=100000000 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"drain_push" --csv --log-file gpurun_out/rlv$v.csv python tools/round_latency.py 4 > /dev/null 2>&1
done
timeout 300 python tools/round_latency.py 20 > gpurun_out/rl_default.json 2>/dev/null
python - <<'PY'
import csv, json
for v in range(4):
    d = json.load(open(f"gpurun_out/rlv{v}.json"))
    rows = list(csv.reader(open(f"gpurun_out/rlv{v}.csv"))); h = None; t = []
    for r in rows:
        if r and r[0] == "ID": h = r; continue
        if h and len(r) == len(h): t.append(round(float(dict(zip(h, r))["Metric Value"].replace(",", "")) / 1000, 1))
    print("variant", v, {k: (x["wall_us"], x["kernel_us"]) for k, x in d.items()}, "ncu", t[1:12:4], t[12:24:4], t[24:36:4], t[36:48:4])
d = json.load(open("gpurun_out/rl_default.json"))
print("default dispatch", {k: (x["wall_us"], x["kernel_us"]) for k, x in d.items()})
PY
