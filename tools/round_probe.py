"""Host cost of a small (decode-pattern) patch round: mark B keys, push, no sync."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2604_12171_b200.perf import PatchRig, Workload
rig = PatchRig(Workload(batch=128, ctx=512))
s = torch.cuda.Stream()
rig.use_stream(s.cuda_stream)
rig.fill()
rig.bulk_round()
torch.cuda.synchronize()
hs = rig.handles
reqs = [h for h in hs for _ in (2, 3)]
grp = [g for _ in hs for g in (2, 3)]
for it in range(3):
    t_mark = t_push = 0.0
    n = 50
    t_all = time.perf_counter()
    for i in range(n):
        t0 = time.perf_counter()
        rig.patch.mark_batch(reqs, grp, [100 + i] * len(reqs), [1] * len(reqs))
        t1 = time.perf_counter()
        rig.patch.push(rig.dst, rig.registry.rank())
        t2 = time.perf_counter()
        t_mark += t1 - t0
        t_push += t2 - t1
    torch.cuda.synchronize()
    print(f"keys/round {len(reqs)}: mark {t_mark/n*1e6:.1f} us, push(host) {t_push/n*1e6:.1f} us, "
          f"per round incl. device {(time.perf_counter()-t_all)/n*1e6:.1f} us")
