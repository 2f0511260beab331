import sys, json
sys.path.insert(0, '.')
import torch
from paper_2604_12171_b200.perf import PatchRig, Workload, c2_live
rig = PatchRig(Workload())
s = torch.cuda.Stream()
rig.use_stream(s.cuda_stream)
rig.fill()
rig.bulk_round()
torch.cuda.synchronize()
print(json.dumps(c2_live(rig, s)))
