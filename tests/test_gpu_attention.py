"""K2 paged-attention decode vs the fp32 numpy oracle (oracle/attention.py).

Tolerance (BASELINE north star), elementwise: |out - ref| <= 2e-2 * |ref| + atol, with
ref the fp32 oracle on the same bf16 K/V/q values and atol = 2^-7 * E_p[|v|] per output
element (oracle/attention.py: the bf16 rounding of P moves an output by ~2^-8 of the
softmax-weighted |v| regardless of the output's own size)."""

import ctypes as C

import numpy as np
import pytest

from oracle.attention import bf16_to_f32, decode_attention

pytestmark = pytest.mark.gpu

RTOL = 2e-2


def _run_case(B, n_q, n_kv, D, s, k, layer, ctxs, seed):
    import torch

    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200 import kvstore

    torch.manual_seed(seed)
    cell = 2 * n_kv * D * 2
    cap = sum((c + s - 1) // s for c in ctxs) + 4
    st = kvstore.KvStore(1, k, s, cap, (0,), cell_bytes=cell)
    kvs = []
    for b, c in enumerate(ctxs):
        x = torch.randn(c, k, 2 * n_kv * D, dtype=torch.bfloat16, device="cuda")
        kvs.append(x)
        if c:
            st.append_seeded(f"att{seed}_{b}", 0, c, 1234 + b, kv_dev=x.data_ptr())
    st.sync()
    rows = torch.tensor([st._registry.handle(f"att{seed}_{b}") for b in range(B)],
                        dtype=torch.int32, device="cuda")
    ctx_t = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    q = torch.randn(B, n_q, D, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    scale = D ** -0.5
    N.check(N.lib().pl_paged_attn_decode(st._h, 0, layer, C.c_void_p(q.data_ptr()),
                                         C.c_void_p(out.data_ptr()), C.c_void_p(rows.data_ptr()),
                                         C.c_void_p(ctx_t.data_ptr()), B, n_q, n_kv, D, scale,
                                         max(ctxs), None))
    torch.cuda.synchronize()
    st.sync()
    qf = bf16_to_f32(q.view(torch.int16).cpu().numpy().view(np.uint16))
    ks, vs = [], []
    for x in kvs:
        u = x[:, layer].view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1, 2, n_kv, D)
        ks.append(bf16_to_f32(u[:, 0]))
        vs.append(bf16_to_f32(u[:, 1]))
    ref, atol = decode_attention(qf, ks, vs, scale, with_atol=True)
    got = bf16_to_f32(out.view(torch.int16).cpu().numpy().view(np.uint16))
    return got, ref, atol


@pytest.mark.parametrize("n_q,n_kv,D", [(32, 8, 128), (64, 8, 128), (8, 8, 128),
                                         (16, 4, 64), (8, 2, 64)])
@pytest.mark.parametrize("s", [8, 16])
def test_decode_matches_fp32_oracle(n_q, n_kv, D, s):
    ctxs = [1, 17, 0, 100, 255, 33, 512, 5]
    got, ref, atol = _run_case(len(ctxs), n_q, n_kv, D, s, 2, 1, ctxs, seed=n_q + D + s)
    err = np.abs(got - ref)
    assert np.all(err <= RTOL * np.abs(ref) + atol), float((err - RTOL * np.abs(ref) - atol).max())
    assert np.all(got[2] == 0)  # empty context -> zeros


def test_decode_long_context_split_k():
    ctxs = [2048, 1999, 4096, 64]
    got, ref, atol = _run_case(len(ctxs), 32, 8, 128, 16, 4, 3, ctxs, seed=7)
    err = np.abs(got - ref)
    assert np.all(err <= RTOL * np.abs(ref) + atol), float((err - RTOL * np.abs(ref) - atol).max())


@pytest.mark.parametrize("ctxs", [[3, 0, 40], [1] * 7, [0, 0, 0], [5000, 1, 1, 1, 900],
                                  [17] * 300])
def test_decode_ragged_schedules(ctxs):
    """stream-K schedule edge cases: fewer stages than CTAs (empty CTA ranges inside a
    sequence), all-empty batches, one long sequence over many CTAs, B > CTAs."""
    got, ref, atol = _run_case(len(ctxs), 32, 8, 128, 16, 1, 0, ctxs, seed=len(ctxs))
    err = np.abs(got - ref)
    assert np.all(err <= RTOL * np.abs(ref) + atol), float((err - RTOL * np.abs(ref) - atol).max())
    for b, c in enumerate(ctxs):
        if c == 0:
            assert np.all(got[b] == 0)


@pytest.mark.parametrize("s,poison", [(16, False), (16, True), (4, True), (8, True)],
                         ids=["mma", "mma_stale_nan_rows", "simt_stale_nan_rows",
                              "mma_8tok_stale_nan_rows"])
def test_decode_raw_entry_over_caller_pool(s, poison):
    """pl_paged_attn_decode_raw: the same kernel over a pool and block table the caller
    owns (a pipeshift integration that keeps its own allocator).  `poison`: every pool
    byte the decode must not use -- rows past each context (which the tensor-core kernel's
    8-token TMA boxes do load), other layers, free units -- is 0xFF (bf16 NaN), as stale
    pool memory can be; the output must still match (s = 4 runs the CUDA-core kernel)."""
    import ctypes as C

    import torch

    from paper_2604_12171_b200 import _native as N

    torch.manual_seed(3)
    B, n_q, n_kv, D, k = 3, 32, 8, 128, 2
    cell = 2 * n_kv * D * 2
    fp = 128
    unit = fp + k * s * cell
    ctxs = [33, 5, 70]
    nb = [(c + s - 1) // s for c in ctxs]
    max_blocks = max(nb)
    slots = torch.randperm(sum(nb) + 3)[: sum(nb)].tolist()   # scattered slots
    pool = torch.full(((sum(nb) + 3) * unit,), 0xFF if poison else 0, dtype=torch.uint8,
                      device="cuda")
    table = torch.full((B, max_blocks), -1, dtype=torch.int32)
    kvs, i = [], 0
    layer = 1
    for b, c in enumerate(ctxs):
        x = torch.randn(c, 2 * n_kv * D, dtype=torch.bfloat16, device="cuda")
        kvs.append(x)
        for j in range(nb[b]):
            table[b, j] = slots[i]
            toks = x[j * s:(j + 1) * s]
            off = slots[i] * unit + fp + layer * s * cell
            pool[off: off + toks.numel() * 2].copy_(toks.contiguous().view(torch.uint8).reshape(-1))
            i += 1
    table = table.cuda()
    ctx_t = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    q = torch.randn(B, n_q, D, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    N.check(N.lib().pl_paged_attn_decode_raw(
        C.c_void_p(pool.data_ptr()), unit, fp, s, k, layer, C.c_void_p(q.data_ptr()),
        C.c_void_p(out.data_ptr()), C.c_void_p(table.data_ptr()), max_blocks,
        C.c_void_p(ctx_t.data_ptr()), B, n_q, n_kv, D, D ** -0.5, max(ctxs), None))
    torch.cuda.synchronize()
    qf = bf16_to_f32(q.view(torch.int16).cpu().numpy().view(np.uint16))
    ks, vs = [], []
    for x in kvs:
        u = x.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1, 2, n_kv, D)
        ks.append(bf16_to_f32(u[:, 0]))
        vs.append(bf16_to_f32(u[:, 1]))
    ref, atol = decode_attention(qf, ks, vs, D ** -0.5, with_atol=True)
    got = bf16_to_f32(out.view(torch.int16).cpu().numpy().view(np.uint16))
    err = np.abs(got - ref)
    assert np.all(err <= RTOL * np.abs(ref) + atol), float((err - RTOL * np.abs(ref) - atol).max())


@pytest.mark.parametrize("n_q", [32, 64])
def test_cuda_core_fallback_for_small_blocks(n_q):
    """4-token blocks are outside the tensor-core kernel's envelope (8-token TMA boxes):
    the CUDA-core kernel serves them, with the same tolerance."""
    ctxs = [1, 17, 0, 100, 255, 33]
    got, ref, atol = _run_case(len(ctxs), n_q, 8, 128, 4, 2, 1, ctxs, seed=n_q)
    err = np.abs(got - ref)
    assert np.all(err <= RTOL * np.abs(ref) + atol), float((err - RTOL * np.abs(ref) - atol).max())
    assert np.all(got[2] == 0)


@pytest.mark.parametrize("n_q", [32, 64], ids=["llama3_8b", "llama3_70b"])
def test_decode_full_bench_shape_sampled(n_q):
    """K2 at the bench's full shape (B = 256, ctx = 2048, 16-token blocks, k = 4, 8 KV heads
    x 128): the whole batch runs as one launch (stream-K over 148 SMs); 16 sampled
    sequences are checked against the fp32 oracle."""
    import torch

    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200 import kvstore

    B, ctx, n_kv, D, s, k, layer = 256, 2048, 8, 128, 16, 4, 2
    torch.manual_seed(n_q)
    cell = 2 * n_kv * D * 2
    st = kvstore.KvStore(1, k, s, B * ctx // s + 8, (0,), cell_bytes=cell)
    pick = sorted(np.random.default_rng(n_q).choice(B, 16, replace=False).tolist())
    keep = {}
    for b in range(B):
        x = torch.randn(ctx, k, 2 * n_kv * D, dtype=torch.bfloat16, device="cuda")
        st.append_seeded(f"full{b}", 0, ctx, 99 + b, kv_dev=x.data_ptr())
        if b in pick:
            keep[b] = x[:, layer].view(torch.int16).cpu().numpy().view(np.uint16)
        st.sync()
        del x
    rows = torch.tensor([st._registry.handle(f"full{b}") for b in range(B)], dtype=torch.int32,
                        device="cuda")
    ctx_t = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    q = torch.randn(B, n_q, D, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    N.check(N.lib().pl_paged_attn_decode(st._h, 0, layer, C.c_void_p(q.data_ptr()),
                                         C.c_void_p(out.data_ptr()), C.c_void_p(rows.data_ptr()),
                                         C.c_void_p(ctx_t.data_ptr()), B, n_q, n_kv, D, D ** -0.5,
                                         ctx, None))
    torch.cuda.synchronize()
    qf = bf16_to_f32(q.view(torch.int16).cpu().numpy().view(np.uint16))[pick]
    ks = [bf16_to_f32(keep[b].reshape(-1, 2, n_kv, D)[:, 0]) for b in pick]
    vs = [bf16_to_f32(keep[b].reshape(-1, 2, n_kv, D)[:, 1]) for b in pick]
    ref, atol = decode_attention(qf, ks, vs, D ** -0.5, with_atol=True)
    got = bf16_to_f32(out.view(torch.int16).cpu().numpy().view(np.uint16))[pick]
    err = np.abs(got - ref)
    assert np.all(err <= RTOL * np.abs(ref) + atol), float((err - RTOL * np.abs(ref) - atol).max())
    st.close()
