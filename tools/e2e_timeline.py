"""Device-busy vs wall time of the pipelined e2e loop (bench.measure_e2e_api shape):
per-kernel CUDA-event time per step next to the wall time per step."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_12171_b200 import _native as N  # noqa: E402
from paper_2604_12171_b200.events import stable_hash  # noqa: E402
from paper_2604_12171_b200.perf import (PatchRig, Workload, append_batch_payloads,  # noqa: E402
                                        engine_payloads)

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
res = torch.zeros(64, dtype=torch.int64, pin_memory=True)


HT = np.zeros(5)


def step(i):
    t = [time.perf_counter()]
    rig.src.free_requests(names)
    t.append(time.perf_counter())
    rig.dst.free_requests(names)
    t.append(time.perf_counter())
    append_batch_payloads(rig.src, reqs, groups, counts, host, mark=True)
    t.append(time.perf_counter())
    rig.patch.push(rig.dst, rig.registry.rank())
    t.append(time.perf_counter())
    N.check(N.lib().pl_patch_device_drained_async(rig.patch.h, C.c_void_p(res.data_ptr() + 8 * i)))
    t.append(time.perf_counter())
    HT[:] += np.diff(t)


for i in range(3):
    step(i)
torch.cuda.synchronize()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
N.check(N.lib().pl_timing_reset())
N.check(N.lib().pl_timing_enable(1))
HT[:] = 0
e_first, e_last = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e_first.record(s)
for i in range(K):
    step(i)
e_last.record(s)
t_enq = time.perf_counter()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K * 1e3
print("device span %.3f ms/step; host enqueue done at %.1f ms, wall %.1f ms"
      % (e_first.elapsed_time(e_last) / K, (t_enq - t0) * 1e3, wall * K))
N.check(N.lib().pl_timing_enable(0))
tot = 0.0
for k in ("kv_write", "drain", "patch_push", "apply_deltas", "partition", "mark"):
    ms, n = N.timing(k)
    if n:
        tot += ms
        print(f"{k:14s} {ms / K:7.3f} ms/step  ({n} launches)")
print(f"timed kernels {tot / K:7.3f} ms/step; wall {wall:7.3f} ms/step")
print("host ms/step: free src %.3f, free dst %.3f, append %.3f, push %.3f, d2h %.3f (sum %.3f)"
      % (*(HT / K * 1e3), HT.sum() / K * 1e3))

# device timeline of one steady step: events on the store stream between the calls
evs = []


def mark():
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    evs.append(e)


for i in range(6):
    mark()
    rig.src.free_requests(names)
    mark()
    rig.dst.free_requests(names)
    mark()
    append_batch_payloads(rig.src, reqs, groups, counts, host, mark=True)
    mark()
    rig.patch.push(rig.dst, rig.registry.rank())
    mark()
torch.cuda.synchronize()
for i in range(1, 6):
    e = evs[5 * i:5 * i + 5]
    nxt = evs[5 * i + 5] if 5 * i + 5 < len(evs) else None
    d = [e[j].elapsed_time(e[j + 1]) for j in range(4)]
    gap = e[4].elapsed_time(nxt) if nxt else float("nan")
    print("step %d device: free src %.3f  free dst %.3f  append %.3f  push %.3f  -> next %.3f ms"
          % (i, *d, gap))
