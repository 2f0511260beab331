"""Time K2 at the bench shape with CUDA events (device time per launch, GB/s)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2604_12171_b200 import _native as N
from paper_2604_12171_b200.perf import Workload, append_batch
from paper_2604_12171_b200.kvstore import KvStore, RequestRegistry
from paper_2604_12171_b200.events import stable_hash

import os
for n_q, n_kv in [(32, 8), (64, 8)]:
    wl = Workload(n_q=n_q, n_kv=n_kv)
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
    def run():
        for j in range(wl.k):
            N.check(N.lib().pl_paged_attn_decode(st._h, 0, j, C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
                    C.c_void_p(rows.data_ptr()), C.c_void_p(ctx_t.data_ptr()), B, wl.n_q, wl.n_kv, wl.head_dim,
                    wl.head_dim ** -0.5, ctx, None))
    for _ in range(3): run()
    torch.cuda.synchronize()
    N.check(N.lib().pl_timing_reset()); N.check(N.lib().pl_timing_enable(1))
    for _ in range(10): run()
    torch.cuda.synchronize()
    ms, n = N.timing("paged_attn")
    N.check(N.lib().pl_timing_enable(0))
    per = ms / n
    gb = B * ctx * wl.cell_bytes / 1e9
    print(f"{'simt' if os.environ.get('PL_ATTN_SIMT') else 'mma'} n_q={n_q} n_kv={n_kv}: {per*1e3:.1f} us/layer  {gb/(per/1e3):.0f} GB/s  ({n} launches)")
    del st
