"""Latency anatomy of one steady patch round (c5_sweep's decode pattern and 1 / 5 / 25 %
random dirty rates, 64 requests x 2048 tokens x 2 k=4 groups, 16-token blocks):
host enqueue time of pl_patch_push, wall time to a synced destination (kernel timing
off), the time until the host bookkeeping worker is idle again, and -- in separate rounds
with kernel timing on -- the device time of the round's kernels.  PL_TRACE_PUSH=1 adds
the push's host phase split on stderr.

    python tools/round_latency.py [rounds]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_12171_b200 import _native as N  # noqa: E402
from paper_2604_12171_b200.events import stable_hash  # noqa: E402
from paper_2604_12171_b200.kvstore import KvStore, RequestRegistry  # noqa: E402
from paper_2604_12171_b200.perf import NativePatch, append_batch, rid  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
batch, ctx, k, s = 64, 2048, 4, 16
reg = RequestRegistry()
blocks = batch * (ctx // s + 1) + 16
src = KvStore(1, k, s, blocks, (0, 1), num_groups=2, cell_bytes=4096, registry=reg)
dst = KvStore(2, k, s, blocks, (0, 1), num_groups=2, cell_bytes=4096, registry=reg)
hs = [reg.handle(rid(i)) for i in range(batch)]
reqs = [h for h in hs for _ in (0, 1)]
groups = [g for _ in hs for g in (0, 1)]
append_batch(src, reqs, groups, [ctx] * len(reqs),
             [stable_hash(rid(i), g) for i in range(batch) for g in (0, 1)])
patch = NativePatch(src, (0, 1), k)
patch.seed()
patch.push(dst, reg.rank())
src.sync()
dst.sync()
rank = reg.rank()
rng = np.random.default_rng(0)
out = {}
for name, r in (("decode", None), ("0.01", 0.01), ("0.05", 0.05), ("0.25", 0.25)):
    host, wall, idle, dev, phases = [], [], [], [], []
    for it in range(2 * rounds + 4):
        timed_kernels = it >= rounds + 2
        if r is None:
            rq, gq, st = reqs, groups, [ctx - 1] * len(reqs)
        else:
            n_keys = int(round(r * batch * 2 * ctx))
            flat = rng.choice(batch * 2 * ctx, size=n_keys, replace=False)
            rq = [hs[x // (2 * ctx)] for x in flat]
            gq = [int((x // ctx) % 2) for x in flat]
            st = [int(x % ctx) for x in flat]
        patch.mark_batch(rq, gq, st, [1] * len(rq))
        src.sync()
        torch.cuda.synchronize()
        if timed_kernels:
            N.check(N.lib().pl_timing_reset())
            N.check(N.lib().pl_timing_enable(1))
        t0 = time.perf_counter()
        patch.push(dst, rank)
        t1 = time.perf_counter()
        dst.sync()          # the destination stream waits on the round's copy (ev_applied)
        t2 = time.perf_counter()
        src.sync()
        patch.dirty_keys()          # any C-ABI call joins the host bookkeeping worker
        t3 = time.perf_counter()
        if timed_kernels:
            N.check(N.lib().pl_timing_enable(0))
            dev.append((N.timing("drain")[0] + N.timing("patch_push")[0]
                        + N.timing("drain_push")[0]) * 1e3)
        elif it >= 2:
            host.append((t1 - t0) * 1e6)
            wall.append((t2 - t0) * 1e6)
            idle.append((t3 - t0) * 1e6)
            phases.append(patch.last_push_stats())
    out[name] = {"keys": len(rq), "host_us": round(float(np.median(host)), 1),
                 "kernel_us": round(float(np.median(dev)), 1),
                 "wall_us": round(float(np.median(wall)), 1),
                 "wall_us_min": round(float(np.min(wall)), 1),
                 "host_idle_us": round(float(np.median(idle)), 1),
                 "host_phases_us": {k: round(1e3 * float(np.median([p[k] for p in phases])), 1)
                                    for k in phases[0] if k not in ("chunked", "async_bookkeeping")},
                 "async_bookkeeping": bool(phases[-1]["async_bookkeeping"])}
print(json.dumps(out, indent=1))
