"""Cold bulk round anatomy (configs[1]): the seed alone (host, wall), the push alone after a
synced seed (host, wall and its phases), and seed + push back to back, each into a fresh
destination.

    python tools/cold_head_probe.py
"""
import sys, time, json
sys.path.insert(0, ".")
import torch
from paper_2604_12171_b200 import _native as N
from paper_2604_12171_b200.kvstore import KvStore
from paper_2604_12171_b200.perf import PatchRig, Workload
wl = Workload(); rig = PatchRig(wl); s = torch.cuda.Stream(); rig.use_stream(s.cuda_stream); rig.fill()
cap = wl.batch * (wl.blocks_per_req + 2) + 64
def fresh():
    rig.dst.close()
    rig.dst = KvStore(2, wl.k, wl.s, cap, (), num_groups=wl.model_groups, cell_bytes=wl.cell_bytes, registry=rig.registry)
    rig.dst.resident_groups |= set(wl.mig_groups)
    N.check(N.lib().pl_store_set_stream(rig.dst._h, N.C.c_void_p(s.cuda_stream)))
    rig.dst.prepare_wait(); torch.cuda.synchronize()
for r in range(6):
    fresh()
    t0 = time.perf_counter(); rig.patch.seed(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    keys, _ = rig.patch.push(rig.dst, rig.registry.rank()); t3 = time.perf_counter(); torch.cuda.synchronize(); t4 = time.perf_counter()
    st = rig.patch.last_push_stats()
    fresh()
    u0 = time.perf_counter(); rig.patch.seed(); rig.patch.push(rig.dst, rig.registry.rank()); u1 = time.perf_counter(); torch.cuda.synchronize(); u2 = time.perf_counter()
    print(json.dumps({"seed_host": round((t1-t0)*1e3,3), "seed_wall": round((t2-t0)*1e3,3), "push_host": round((t3-t2)*1e3,3), "push_wall": round((t4-t2)*1e3,3), "both_host": round((u1-u0)*1e3,3), "both_wall": round((u2-u0)*1e3,3), "pre": st["k3_enqueue"], "reserve": st["reserve"], "flush": st["dst_flush"], "launch": st["copy_enqueue"]}))
