"""Cross-GPU push in one process (needs >= 2 GPUs): source store on cuda:0, destination on
cuda:1; times the fused push (GB/s over NVLink) and, under
`ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum -k regex:"push_batched|copy_kernel"`,
gives the link bytes per launch.  Prints a JSON line; exits 0 with a note on one GPU."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_12171_b200.events import stable_hash  # noqa: E402
from paper_2604_12171_b200.kvstore import KvStore, RequestRegistry  # noqa: E402
from paper_2604_12171_b200.perf import NativePatch, Workload, append_batch, rid  # noqa: E402

if torch.cuda.device_count() < 2:
    print(json.dumps({"skipped": "needs 2 GPUs", "gpus": torch.cuda.device_count()}))
    sys.exit(0)
wl = Workload(batch=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
reg = RequestRegistry()
cap = wl.batch * (wl.blocks_per_req + 2) + 64
src = KvStore(1, wl.k, wl.s, cap, wl.src_groups, num_groups=wl.model_groups,
              cell_bytes=wl.cell_bytes, device=0, registry=reg)
dst = KvStore(2, wl.k, wl.s, cap, (), num_groups=wl.model_groups, cell_bytes=wl.cell_bytes,
              device=1, registry=reg)
dst.resident_groups |= set(wl.mig_groups)
hs = [reg.handle(rid(i)) for i in range(wl.batch)]
append_batch(src, [h for h in hs for _ in wl.src_groups], [g for _ in hs for g in wl.src_groups],
             [wl.ctx] * (len(hs) * len(wl.src_groups)),
             [stable_hash(rid(i), g) for i in range(wl.batch) for g in wl.src_groups])
src.sync()
p = NativePatch(src, wl.mig_groups, wl.k)
times = []
for it in range(4):
    p.seed()
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    t0 = time.perf_counter()
    keys, cells = p.push(dst, reg.rank())
    src.sync()
    dst.sync()
    times.append(time.perf_counter() - t0)
payload = cells * wl.cell_bytes
t = sorted(times[1:])[len(times[1:]) // 2]
print(json.dumps({"payload_bytes": payload, "ms": round(t * 1e3, 3),
                  "gbs": round(payload / t / 1e9, 1), "peak_nvlink_gbs": 900.0,
                  "frac": round(payload / t / 1e9 / 900.0, 4)}))
