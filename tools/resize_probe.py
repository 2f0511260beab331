"""Resize-latency breakdown on the bench workload (PL_TRACE_RESIZE=1 prints phases)."""
import os
import sys
import time

os.environ.setdefault("PL_TRACE_RESIZE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2604_12171_b200.perf import PatchRig, Workload

wl = Workload()
rig = PatchRig(wl, device=0)
stream = torch.cuda.Stream()
rig.use_stream(stream.cuda_stream)
t0 = time.perf_counter()
rig.fill()
torch.cuda.synchronize()
print(f"fill {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
rig.bulk_round()
torch.cuda.synchronize()
print(bench.measure_resize(rig, stream, torch, wl), flush=True)
