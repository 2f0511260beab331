"""Wall time of parity-mode runs (reference event clock, GPU data plane) for the golden
scenarios; compare with profiles/reference_cpu_r1.json["simulations"] (the reference)."""
import json
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import sim_scenarios  # noqa: E402

from paper_2604_12171_b200.simulation import Simulation  # noqa: E402

out = {}
import torch  # noqa: E402

torch.zeros(1, device="cuda")   # CUDA context outside the timings
for name in ("fig3_seed5", "fig3_seed5", "hetero_c10_seed123", "hetero_n60_seed7"):
    scen, seed, fill = sim_scenarios.golden_runs()[name]
    t0 = time.perf_counter()
    sim = Simulation(scen, seed=seed)
    if fill:
        fill(sim)
    sim.scheduler.run(until=600.0)
    out[name + ("" if name not in out else "_again")] = {"seconds": round(time.perf_counter() - t0, 3), "events": len(sim.trace)}
print(json.dumps(out))
