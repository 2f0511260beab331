"""Standalone driver for profiling K2 (and K1) at the bench shape: B=256, ctx=2048, 1 group."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2604_12171_b200 import _native as N
from paper_2604_12171_b200.perf import Workload, append_batch
from paper_2604_12171_b200.kvstore import KvStore, RequestRegistry
from paper_2604_12171_b200.events import stable_hash

import os
wl = Workload(n_q=int(os.environ.get("PL_NQ", "32")))
reg = RequestRegistry()
B, ctx = wl.batch, wl.ctx
st = KvStore(1, wl.k, wl.s, B * (wl.blocks_per_req + 1), (0,), num_groups=8, cell_bytes=wl.cell_bytes, registry=reg)
hs = [reg.handle(f"r{i}") for i in range(B)]
append_batch(st, hs, [0] * B, [ctx] * B, [stable_hash(f"r{i}", 0) for i in range(B)])
st.sync()
rows = torch.tensor(hs, dtype=torch.int32, device="cuda")
ctx_t = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
q = torch.randn(B, wl.n_q, wl.head_dim, dtype=torch.bfloat16, device="cuda")
out = torch.empty_like(q)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    for j in range(wl.k):
        N.check(N.lib().pl_paged_attn_decode(st._h, 0, j, C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
                C.c_void_p(rows.data_ptr()), C.c_void_p(ctx_t.data_ptr()), B, wl.n_q, wl.n_kv, wl.head_dim,
                wl.head_dim ** -0.5, ctx, None))
torch.cuda.synchronize()
print("ok")
