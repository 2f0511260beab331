"""Anatomy of the cold bulk round (value_cold): the first drain + push of configs[1]'s
migrating groups into a destination with no chains yet.  Each rep makes a fresh
destination store, optionally waits for its lazily mapped pools (as Phase 3 does before
the bulk patch), then times seed + push to a synced destination and prints the push's host
phases (pl_patch_last_push_stats) and the copy's device time.

    python tools/cold_probe.py [reps] [wait_pools=1]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2604_12171_b200 import _native as N  # noqa: E402
from paper_2604_12171_b200.kvstore import KvStore  # noqa: E402
from paper_2604_12171_b200.perf import PatchRig, Workload  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wait_pools = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
wl = Workload()
rig = PatchRig(wl)
s = torch.cuda.Stream()
rig.use_stream(s.cuda_stream)
rig.fill()
torch.cuda.synchronize()
cap = wl.batch * (wl.blocks_per_req + 2) + 64
out = []
for r in range(reps):
    if r:
        rig.dst.close()
        rig.dst = KvStore(2, wl.k, wl.s, cap, (), num_groups=wl.model_groups,
                          cell_bytes=wl.cell_bytes, registry=rig.registry)
        rig.dst.resident_groups |= set(wl.mig_groups)
        N.check(N.lib().pl_store_set_stream(rig.dst._h, N.C.c_void_p(s.cuda_stream)))
    tw = time.perf_counter()
    waited = rig.dst.prepare_wait() if wait_pools else 0.0
    tw = (time.perf_counter() - tw) * 1e3
    torch.cuda.synchronize()
    N.check(N.lib().pl_timing_reset())
    N.check(N.lib().pl_timing_enable(1))
    t0 = time.perf_counter()
    keys, _ = rig.bulk_round()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    N.check(N.lib().pl_timing_enable(0))
    st = rig.patch.last_push_stats()
    push_ms, push_n = N.timing("patch_push")
    out.append({"rep": r, "pools_wait_ms": round(tw, 3), "keys": keys,
                "host_ms": round((t1 - t0) * 1e3, 3), "wall_ms": round((t2 - t0) * 1e3, 3),
                "gbs": round(wl.payload_bytes / (t2 - t0) / 1e9, 1),
                "copy_device_ms": round(push_ms, 3), "copy_launches": push_n,
                "drain_ms": round(N.timing("drain")[0], 3), "phases_ms": st})
    print(json.dumps(out[-1]), flush=True)
