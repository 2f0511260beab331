"""Wall time of the packaged heterogeneous_shift scenario through this package's
parity-mode Simulation (reference clock, GPU data plane)."""
import sys, time, json, hashlib
sys.path.insert(0, '.')
import paper_2604_12171_b200 as ps
sc = ps.load_scenario(sys.argv[1] if len(sys.argv) > 1 else "tests/golden/heterogeneous_shift.yaml")
t0 = time.perf_counter()
res = ps.run_scenario(sc, seed=0)
dt = time.perf_counter() - t0
print(json.dumps({"seconds": round(dt, 2), "events": len(res.trace),
                  "trace_sha": hashlib.sha256(res.trace.to_jsonl().encode()).hexdigest()}))
