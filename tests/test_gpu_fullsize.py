"""Parity at BASELINE configs[1]'s full size (Llama-3-8B shape, B = 256 x 2048 tokens,
4096 B cells, 17.2 GB per bulk round) through size-independent properties: every
fingerprint of both migrating groups on the destination equals the source's and the
engine's payload (engine.py:252-261); sampled cells are bit-exact copies and equal the
oracle's expansion of their fingerprint; a steady round after random writes moves exactly
the marked keys; the pipelined cold push (runs) and the one-launch push give identical
destinations (same block ids).  Beyond samples, every live cell of every store is
checked on the device (csrc/verify.cu): all 4096 B of every cell against the expansion
of its fingerprint, every fingerprint against the engine payload, and the destination
against the source byte for byte."""

import random

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _rig(chunked, monkeypatch):
    from paper_2604_12171_b200.perf import PatchRig, Workload
    if chunked:
        monkeypatch.delenv("PL_PUSH_NO_CHUNK", raising=False)
    else:
        monkeypatch.setenv("PL_PUSH_NO_CHUNK", "1")
    rig = PatchRig(Workload())
    rig.fill()
    return rig


def _full_check(rig):
    """Every live cell of both stores, on the device: all bytes = the expansion of the
    cell's fingerprint, every fingerprint = the engine payload of its position; and the
    destination's migrating groups = the source's, byte for byte (csrc/verify.cu)."""
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import rid
    wl = rig.wl
    seeds = {(rid(i), g): stable_hash(rid(i), g) for i in range(wl.batch) for g in wl.src_groups}
    live = sum(len(rig.src.tables[rid(i)].chain) for i in range(wl.batch))
    v = rig.src.verify_cells(seeds)
    assert v["bad_bytes"] == 0 and v["bad_fingerprints"] == 0 and v["first_bad"] == -1, v
    written = sum(rig.src.tables[rid(i)].written[g] for i in range(wl.batch) for g in wl.src_groups)
    assert v["cells"] == written and live > 0
    d = rig.dst.verify_cells(seeds)
    assert d["bad_bytes"] == 0 and d["bad_fingerprints"] == 0, d
    mig = sum(rig.src.tables[rid(i)].written[g] for i in range(wl.batch) for g in wl.mig_groups)
    assert d["cells"] == mig
    c = rig.src.compare_cells(rig.dst, wl.mig_groups)
    assert c["bad_positions"] == 0 and c["missing"] == 0 and c["cells"] == mig * wl.k, c
    return v["cells"] + d["cells"]


def _check_group(rig, g, rng, n_samples=64):
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import engine_payloads, rid
    wl = rig.wl
    src, dst = rig.src.snapshot_group(g), rig.dst.snapshot_group(g)
    assert len(dst) == wl.batch and dst == src
    for i in rng.sample(range(wl.batch), 8):          # fingerprints = the engine's payloads
        want = engine_payloads(stable_hash(rid(i), g), len(dst[rid(i)]))
        assert np.array_equal(np.array(dst[rid(i)], dtype=np.uint64), want)
    for _ in range(n_samples):                        # bytes: copy of the source, = expansion
        i, pos, j = rng.randrange(wl.batch), rng.randrange(wl.ctx), rng.randrange(wl.k)
        cell = rig.dst.read_cell(rid(i), g, pos, j)
        assert cell == rig.src.read_cell(rid(i), g, pos, j)
        assert cell == oracle.expand_cell(dst[rid(i)][pos], j, wl.cell_bytes)


@pytest.fixture(scope="module")
def runs():
    return {}


@pytest.mark.parametrize("chunked", [True, False])
def test_fullsize_bulk_round(monkeypatch, runs, chunked):
    import torch
    rng = random.Random(7)
    rig = _rig(chunked, monkeypatch)
    torch.cuda.synchronize()
    keys, cells = rig.bulk_round()
    rig.src.sync()
    rig.dst.sync()
    wl = rig.wl
    assert keys == wl.batch * wl.ctx * len(wl.mig_groups)
    assert cells * wl.cell_bytes == wl.payload_bytes == 17_179_869_184
    for g in wl.mig_groups:
        _check_group(rig, g, rng)
    # every byte: 17.2 GB patched + 34.4 GB of source cells, on the device
    assert _full_check(rig) == wl.batch * wl.ctx * (len(wl.src_groups) + len(wl.mig_groups))
    # block ids of the destination chains: identical with and without the pipelined runs
    from paper_2604_12171_b200.perf import rid
    runs[chunked] = [[b.block_id for b in rig.dst.tables[rid(i)].chain] for i in range(0, wl.batch, 17)]
    if len(runs) == 2:
        assert runs[True] == runs[False]
    rig.destroy()


def test_fullsize_steady_round_moves_exactly_the_marked_keys(monkeypatch):
    """After the bulk round, append one token to a random half of the requests in both
    migrating groups (K1 with the fused dirty mark): the next round drains exactly those
    keys and the destination again equals the source."""
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import append_batch, rid
    rng = random.Random(11)
    rig = _rig(True, monkeypatch)
    rig.bulk_round()
    wl = rig.wl
    pick = sorted(rng.sample(range(wl.batch), wl.batch // 2))
    reqs = [rig.handles[i] for i in pick for _ in wl.src_groups]
    groups = [g for _ in pick for g in wl.src_groups]
    append_batch(rig.src, reqs, groups, [1] * len(reqs),
                 [stable_hash(rid(i), g) for i in pick for g in wl.src_groups], mark=True)
    keys, _ = rig.patch.push(rig.dst, rig.registry.rank())
    rig.src.sync()
    rig.dst.sync()
    assert keys == len(pick) * len(wl.mig_groups)
    for g in wl.mig_groups:
        _check_group(rig, g, rng, n_samples=16)
        for i in pick[:8]:                            # the new token is there, bit-exact
            assert rig.dst.read_cell(rid(i), g, wl.ctx, 0) == rig.src.read_cell(rid(i), g, wl.ctx, 0)
    _full_check(rig)
    # more steady rounds, including requests that finish mid-migration
    for step in range(3):
        pick = sorted(rng.sample(range(wl.batch), wl.batch // 4))
        reqs = [rig.handles[i] for i in pick for _ in wl.src_groups]
        groups = [g for _ in pick for g in wl.src_groups]
        append_batch(rig.src, reqs, groups, [1 + step] * len(reqs),
                     [stable_hash(rid(i), g) for i in pick for g in wl.src_groups], mark=True)
        rig.patch.push(rig.dst, rig.registry.rank())
    rig.src.sync()
    rig.dst.sync()
    _full_check(rig)
    rig.destroy()


def test_fullsize_configs2_live_resize():
    """BASELINE configs[2] (Llama-3-70B shape, PP 4 -> 8, HBM pre-filled to ~100 GB of live
    KV): Phase-2 shrink relocates >13 k live blocks with K6, the leaving groups are patched
    to a destination, then dropped, and the stage grows to b_new.  Sampled fingerprints and
    4096-B cells survive every step; the destination's groups equal the source's."""
    import gc

    import torch

    from paper_2604_12171_b200.perf import c3_live_resize
    gc.collect()
    torch.cuda.empty_cache()
    out = c3_live_resize(0, check=True)
    assert out["checks"] == ["relocation", "patched(dst)", "drop+grow"]
    # every live cell, not samples: after the K6 relocation, the patch, the drop + grow
    full = out["full_checks"]
    assert [f["what"] for f in full] == ["relocation", "patched", "patched(dst)", "drop+grow"]
    for f in full:
        assert f["bad"] == 0 and f["cells"] > 0, f
    # 76 k live blocks x 16 tokens x 5 groups token-cells (x 4 layers x 4096 B = 100 GB)
    assert full[0]["cells"] > 6e6 and full[1]["cells"] > 9e6
    assert out["phase2_shrink_stats"]["relocated_blocks"] > 13_000
    assert out["bulk_patch"]["payload_bytes"] > 39e9


def test_max_size_pool_8b_pp8():
    """Maximum size: one Llama-3-8B PP8 stage at the reference budget, max_blocks = 611,320
    blocks of 16 tokens x k = 4 layers x 4096 B (160 GB of KV in one pool, SURVEY §8 sizes).
    Fill every block through K1, then: one more token overflows atomically; sampled
    fingerprints and cells are exact; freeing half the requests and shrinking to half the
    capacity relocates the live blocks above the line (K6) without changing a byte."""
    import gc
    import random

    import torch

    from paper_2604_12171_b200.cluster import GpuSpec, ModelSpec, max_blocks
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.kvstore import KvOverflow, KvStore, RequestRegistry
    from paper_2604_12171_b200.perf import append_batch, engine_payloads, rid

    gc.collect()
    torch.cuda.empty_cache()
    gran = 16 * 4096 * 4
    gpu = GpuSpec(1, 180 * 10 ** 9 // gran * gran, 8e12, 1e-6, 1e-6, gran)
    cap = max_blocks(gpu, 4, ModelSpec(32, 436_000_000, 4096, 4), 0.9)
    assert 600_000 < cap < 620_000
    if torch.cuda.mem_get_info()[0] < cap * (16 * 4 * 4096 + 128) + (4 << 30):
        pytest.skip("needs ~165 GB of free HBM")
    reg = RequestRegistry()
    st = KvStore(1, 4, 16, cap, (0,), num_groups=8, cell_bytes=4096, registry=reg)
    tokens = cap * 16
    n_req = -(-tokens // 2048)
    lens = [2048] * (n_req - 1) + [tokens - 2048 * (n_req - 1)]
    hs = [reg.handle(rid(i)) for i in range(n_req)]
    for c0 in range(0, n_req, 512):
        sl = range(c0, min(n_req, c0 + 512))
        append_batch(st, [hs[i] for i in sl], [0] * len(sl), [lens[i] for i in sl],
                     [stable_hash(rid(i), 0) for i in sl])
    st.sync()
    assert st.used_blocks == cap and st.free_blocks == 0
    with pytest.raises(KvOverflow):
        st.append(rid(0), 0, 1, [1])
    assert st.used_blocks == cap and st.tables[rid(0)].written[0] == 2048
    # every one of the 9.78 M cells (160 GB): bytes = expansion, fingerprint = engine payload
    seeds = {(rid(i), 0): stable_hash(rid(i), 0) for i in range(n_req)}
    v = st.verify_cells(seeds)
    assert v == {"cells": tokens, "bad_bytes": 0, "bad_fingerprints": 0, "first_bad": -1}, v

    rng = random.Random(5)
    keep = [i for i in range(n_req) if i % 2 == 1]
    samples = []
    for _ in range(48):
        i = rng.choice(keep)
        pos, j = rng.randrange(lens[i]), rng.randrange(4)
        fp = int(engine_payloads(stable_hash(rid(i), 0), pos + 1)[pos])
        assert st.read_checksum(rid(i), 0, pos) == fp
        cell = st.read_cell(rid(i), 0, pos, j)
        assert cell == oracle.expand_cell(fp, j, 4096)
        samples.append((i, pos, j, fp, cell))
    st.free_requests([rid(i) for i in range(n_req) if i % 2 == 0])
    live = st.used_blocks
    st.compact()
    st.resize(cap // 2 + 64)
    st.sync()
    assert st.used_blocks == live and st.last_resize_stats()["relocated_blocks"] > 100_000
    for i, pos, j, fp, cell in samples:
        assert st.read_checksum(rid(i), 0, pos) == fp
        assert st.read_cell(rid(i), 0, pos, j) == cell
    v = st.verify_cells({k: sd for k, sd in seeds.items() if int(k[0][1:]) % 2 == 1})
    assert v["bad_bytes"] == 0 and v["bad_fingerprints"] == 0
    assert v["cells"] == sum(lens[i] for i in keep)
    st.close()
