"""Standalone driver for profiling the fused push (K3 + K4/K5) on a bench-shaped pair at a
smaller batch (ncu --set full replays each launch ~40x with memory save/restore)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_12171_b200.perf import PatchRig, Workload  # noqa: E402

rig = PatchRig(Workload(batch=int(sys.argv[1]) if len(sys.argv) > 1 else 32))
rig.fill()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    rig.bulk_round()
torch.cuda.synchronize()
print("ok")
