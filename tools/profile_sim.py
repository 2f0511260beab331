import cProfile, pstats, sys, io
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
torch.zeros(1, device="cuda")
import sim_scenarios
from paper_2604_12171_b200.simulation import Simulation
scen, seed, fill = sim_scenarios.golden_runs()["hetero_n60_seed7"]
pr = cProfile.Profile()
pr.enable()
sim = Simulation(scen, seed=seed)
sim.scheduler.run(until=600.0)
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
