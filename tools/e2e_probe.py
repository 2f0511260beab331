"""Phase breakdown of one e2e step (bench.measure_e2e_api)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2604_12171_b200.perf import PatchRig, Workload, append_batch_payloads, engine_payloads
from paper_2604_12171_b200.events import stable_hash
rig = PatchRig(Workload())
s = torch.cuda.Stream()
rig.use_stream(s.cuda_stream)
wl = rig.wl
names = [f"api{i:04d}" for i in range(wl.batch)]
handles = [rig.registry.handle(n) for n in names]
reqs = [h for h in handles for _ in wl.mig_groups]
groups = [g for _ in handles for g in wl.mig_groups]
counts = [wl.ctx] * len(reqs)
host = np.concatenate([engine_payloads(stable_hash(n, g), wl.ctx) for n in names for g in wl.mig_groups])
for it in range(4):
    t = [time.perf_counter()]
    rig.src.free_requests(names); rig.dst.free_requests(names)
    t.append(time.perf_counter())
    append_batch_payloads(rig.src, reqs, groups, counts, host, mark=True)
    t.append(time.perf_counter())
    keys, _ = rig.patch.push(rig.dst, rig.registry.rank())
    t.append(time.perf_counter())
    d = rig.patch.device_drained()
    t.append(time.perf_counter())
    print("free %.2f  append(host) %.2f  push(host) %.2f  wait+D2H %.2f ms" % tuple((b - a) * 1e3 for a, b in zip(t, t[1:])))
