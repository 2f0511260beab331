import sys, json
sys.path.insert(0, '.')
import torch
from paper_2604_12171_b200.perf import PatchRig, Workload, c2_live
from paper_2604_12171_b200 import _native as N
rig = PatchRig(Workload())
s = torch.cuda.Stream()
rig.use_stream(s.cuda_stream)
rig.fill()
rig.bulk_round()
torch.cuda.synchronize()
N.check(N.lib().pl_timing_reset()); N.check(N.lib().pl_timing_enable(1))
print(json.dumps(c2_live(rig, s)))
for k in ("patch_push", "paged_attn", "kv_write"):
    print(k, N.timing(k))
