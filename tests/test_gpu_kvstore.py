"""GPU block manager parity: the CUDA-backed KvStore replays the reference's
own op sequences (tests/golden/kv_sequences.json) and must match them, and the
oracle, bit for bit: results, counters, block order, chains, fingerprints,
state digest.  Mirrors pkg/tests/test_kvstore.py of the reference."""

import hashlib

import numpy as np
import pytest

import opgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kv():
    from paper_2604_12171_b200 import kvstore
    return kvstore


@pytest.mark.parametrize("seed", range(40))
def test_gpu_store_replays_reference(kv, golden, seed):
    case = golden("kv_sequences.json")[seed]
    p = case["params"]
    st = kv.KvStore(p["gpu_id"], p["k"], p["s"], p["capacity"], p["groups"], cell_bytes=64)
    ref = oracle.OracleStore(p["gpu_id"], p["k"], p["s"], p["capacity"], p["groups"], cell_bytes=64)
    excs = (kv.KvError, ValueError)
    for i, op in enumerate(opgen.kv_ops(seed)):
        got = opgen.apply_op(st, op, excs)
        assert got == case["results"][i], (i, op)
        assert opgen.apply_op(ref, op, (oracle.KvError, ValueError)) == got
        assert opgen.light_state(st) + [st.occupied_cells] == case["lights"][i], (i, op)
    assert opgen.full_state(st) == case["final"]
    assert hashlib.sha256(repr(st.state_digest()).encode()).hexdigest() == case["digest_sha"]
    # the KV bytes behind every fingerprint are the deterministic expansion (oracle)
    for rid in sorted(st.tables):
        for g, w in st.tables[rid].written.items():
            for pos in range(0, w, max(1, w // 5)):
                try:
                    fp = st.read_checksum(rid, g, pos)
                except kv.UnknownSlot:
                    continue
                for j in range(p["k"]):
                    assert st.read_cell(rid, g, pos, j) == oracle.expand_cell(fp, j, 64)
                    assert ref.read_cell(rid, g, pos, j) == st.read_cell(rid, g, pos, j)


class TestReferenceUnitCases:
    """The reference's known answers (pkg/tests/test_kvstore.py)."""

    def store(self, kv, capacity=10, s=16, k=4, groups=(0,)):
        return kv.KvStore(1, k, s, capacity, groups)

    def fill(self, st, rid, g, n):
        start = st.tables[rid].written.get(g, 0) if rid in st.tables else 0
        return st.append(rid, g, n, [opgen.payload(rid, g, start + i) for i in range(n)])

    def test_forty_tokens_three_blocks(self, kv):
        st = self.store(kv)
        slots = self.fill(st, "r1", 0, 40)
        assert st.used_blocks == 3
        assert [s.offset for s in slots] == list(range(16)) * 2 + list(range(8))
        assert [s.block_id for s in slots] == [0] * 16 + [1] * 16 + [2] * 8

    def test_overflow_atomic(self, kv):
        st = self.store(kv, capacity=2)
        self.fill(st, "r1", 0, 20)
        with pytest.raises(kv.KvOverflow):
            self.fill(st, "r2", 0, 40)
        assert st.used_blocks == 2 and "r2" not in st.tables

    def test_lookup_token_20(self, kv):
        st = self.store(kv)
        self.fill(st, "r1", 0, 25)
        addr, off = st.lookup("r1", 1, 20)
        assert off == 4 and addr == st.tables["r1"].chain[1].address

    def test_compaction_partition_and_survival(self, kv):
        st = self.store(kv, capacity=5)
        for r in "abcde":
            self.fill(st, r, 0, 16)
        st.free_request("b")
        st.free_request("d")
        before = {(r, p): st.lookup(r, 1, p) for r in "ace" for p in range(16)}
        assert st.compact() == 2
        assert [b.state for b in st.blocks] == ["live"] * 3 + ["free"] * 2
        for (r, p), v in before.items():
            assert st.lookup(r, 1, p) == v
            assert st.read_checksum(r, 0, p) == opgen.payload(r, 0, p)

    def test_resize_relocates_live_units_and_releases_memory(self, kv):
        # live blocks sitting in the physical tail are moved by K6 so the pool's tail
        # can be unmapped; every fingerprint and byte survives
        st = kv.KvStore(1, 2, 16, 64, (0, 1), cell_bytes=4096, chunk_bytes=2 << 20)
        for i in range(40):
            self.fill(st, f"x{i}", i % 2, 16)
        for i in range(0, 38):
            st.free_request(f"x{i}")
        keep = ["x38", "x39"]
        before = {(r, p): st.read_cell(r, int(r[1:]) % 2, p, 1) for r in keep for p in range(16)}
        mapped0 = st.info()["mapped_bytes"]
        st.resize(4)
        stats = st.last_resize_stats()
        assert st.capacity_blocks == 4 and stats["relocated_blocks"] == 2
        assert stats["bytes_unmapped"] > 0 and st.info()["mapped_bytes"] < mapped0
        for (r, p), v in before.items():
            assert st.read_cell(r, int(r[1:]) % 2, p, 1) == v
            assert st.read_checksum(r, int(r[1:]) % 2, p) == opgen.payload(r, int(r[1:]) % 2, p)
        st.resize(64)
        assert st.info()["mapped_bytes"] >= mapped0
        self.fill(st, "y", 0, 16 * 60)
        assert st.used_blocks == 62

    def test_drop_one_group_keeps_shared_blocks(self, kv):
        st = self.store(kv, capacity=8, groups=(0, 1))
        self.fill(st, "a", 0, 32)
        self.fill(st, "a", 1, 32)
        occ = sum(b.occupied_tokens() for b in st.blocks)
        assert st.drop_layer_groups([0]) == 32
        assert st.used_blocks == 2
        assert st.read_checksum("a", 1, 17) == opgen.payload("a", 1, 17)
        assert sum(b.occupied_tokens() for b in st.blocks) == occ // 2
        with pytest.raises(kv.UnknownLayerGroup):
            st.drop_layer_groups([3])

    def test_utilization_quarter_block(self, kv):
        st = kv.KvStore(1, 4, 64, 4, (0,))
        self.fill(st, "a", 0, 16)
        assert st.effective_utilization() == 0.25

    def test_seeded_append_matches_engine_payloads(self, kv, golden):
        st = self.store(kv)
        seed = opgen.stable_hash("r0000", 0)
        st.append_seeded("r0000", 0, 4, seed)
        got = [st.read_checksum("r0000", 0, p) for p in range(4)]
        assert got == golden("fingerprints.json")["engine_r0000_g0"]


class TestDeferredReclaim:
    """Physical reclaim off the critical path (vmm.cu): a shrink retires its tail
    chunks, a grow inside the grace period takes them back still mapped, a forced
    reclaim returns every byte to the driver, and the live KV never changes."""

    def test_shrink_grow_reuse_and_reclaim(self, kv):
        gran = 2 << 20
        # 16-token blocks of 4 x 4096 B cells: 256 KiB + header per unit, 8 units per chunk
        st = kv.KvStore(1, 4, 16, 64, (0, 1), cell_bytes=4096, chunk_bytes=gran)
        for i in range(40):
            st.append_seeded(f"x{i}", i % 2, 16, 1000 + i)
        for i in range(0, 38):
            st.free_request(f"x{i}")
        keep = ["x38", "x39"]
        before = {(r, p): st.read_cell(r, int(r[1:]) % 2, p, 3) for r in keep for p in (0, 7, 15)}
        v0 = st.vmm_stats()
        mapped0 = st.info()["mapped_bytes"]
        st.resize(4)
        assert st.info()["mapped_bytes"] < mapped0
        assert st.vmm_stats()["pending_reclaim_bytes"] > 0
        # grow back at once: the retired tail is still mapped and is taken back as is
        st.resize(64)
        v1 = st.vmm_stats()
        assert v1["tail_reused_chunks"] > v0["tail_reused_chunks"]
        assert v1["created_chunks"] == v0["created_chunks"]
        assert st.info()["mapped_bytes"] >= mapped0
        for (r, p), v in before.items():
            assert st.read_cell(r, int(r[1:]) % 2, p, 3) == v
        # shrink, force the reclaim, grow: fresh chunks from the driver
        st.resize(4)
        st.reclaim()
        assert st.vmm_stats()["pending_reclaim_bytes"] == 0
        st.resize(64)
        v2 = st.vmm_stats()
        assert v2["created_chunks"] > v1["created_chunks"]
        for (r, p), v in before.items():
            assert st.read_cell(r, int(r[1:]) % 2, p, 3) == v
        st.append_seeded("y", 0, 16 * 60, 7)
        assert st.read_checksum("y", 0, 16 * 60 - 1) == oracle.payload(7, 16 * 60 - 1)

    def test_drop_group_releases_in_background(self, kv):
        st = kv.KvStore(1, 4, 16, 32, (0, 1), cell_bytes=4096, chunk_bytes=2 << 20)
        for i in range(8):
            st.append_seeded(f"a{i}", 0, 40, i)
            st.append_seeded(f"a{i}", 1, 40, 100 + i)
        keep = {p: st.read_cell("a3", 1, p, 2) for p in (0, 39)}
        st.drop_layer_groups([0])
        assert st.vmm_stats()["pending_reclaim_bytes"] > 0
        st.reclaim()
        assert st.vmm_stats()["pending_reclaim_bytes"] == 0
        for p, v in keep.items():
            assert st.read_cell("a3", 1, p, 2) == v
        # the dropped group can come back (fresh reservation) and be written again
        st.resident_groups.add(0)
        st.append_seeded("b", 0, 20, 5)
        assert st.read_cell("a3", 1, 39, 2) == keep[39]

    def test_store_teardown_with_pending_reclaim(self, kv):
        for _ in range(3):
            st = kv.KvStore(1, 2, 16, 64, (0,), cell_bytes=4096, chunk_bytes=2 << 20)
            st.append_seeded("a", 0, 100, 1)
            st.resize(8)
            del st


def test_free_requests_batch_equals_one_by_one():
    from paper_2604_12171_b200 import kvstore as kv
    from paper_2604_12171_b200.events import stable_hash

    stores = []
    for _ in range(2):
        reg = kv.RequestRegistry()
        st = kv.KvStore(1, 2, 16, 256, (0, 1), cell_bytes=64, registry=reg)
        for i in range(20):
            for g in (0, 1):
                st.append_seeded(f"q{i}", g, 5 + 9 * i, stable_hash(f"q{i}", g))
        stores.append(st)
    gone = [f"q{i}" for i in range(0, 20, 3)] + ["never-seen"]
    for r in gone:
        stores[0].free_request(r)
    stores[1].free_requests(gone)
    assert repr(stores[0].state_digest()) == repr(stores[1].state_digest())
    assert stores[0].used_blocks == stores[1].used_blocks
    stores[0].append_seeded("new", 0, 40, 1)
    stores[1].append_seeded("new", 0, 40, 1)
    assert stores[0].tables["new"].chain[0].block_id == stores[1].tables["new"].chain[0].block_id


def test_prepare_grow_creates_the_chunks_ahead():
    """prepare_grow maps the tail a planned grow needs on the reclaimer thread (cached
    chunks first, then new ones); the grow then only adopts it: no cuMemCreate, no map on
    the critical path; KV survives."""
    from paper_2604_12171_b200 import kvstore as kv

    st = kv.KvStore(1, 2, 16, 64, (0, 1, 2), cell_bytes=4096, chunk_bytes=2 << 20)
    for i in range(6):
        st.append_seeded(f"a{i}", 0, 50, i)
        st.append_seeded(f"a{i}", 2, 50, 10 + i)
    keep = st.read_cell("a4", 0, 49, 1)
    asked = st.prepare_grow(256, (0, 2))
    assert asked > 0
    st.prepare_wait()
    v0 = st.vmm_stats()
    st.drop_layer_groups([1])
    st.resize(256)
    v1 = st.vmm_stats()
    assert v1["created_chunks"] == v0["created_chunks"]
    assert v1["tail_reused_chunks"] - v0["tail_reused_chunks"] >= asked
    assert st.read_cell("a4", 0, 49, 1) == keep
    st.append_seeded("big", 2, 16 * 200, 3)


def test_prepare_grow_then_shrink_or_teardown():
    """A prepared (mapped, not yet adopted) tail is adopted by a shrink and retired with
    the rest of the tail; a store torn down with a prepared tail releases it."""
    from paper_2604_12171_b200 import kvstore as kv

    st = kv.KvStore(1, 2, 16, 64, (0, 1), cell_bytes=4096, chunk_bytes=2 << 20)
    st.append_seeded("a", 0, 300, 1)
    keep = st.read_cell("a", 0, 299, 1)
    assert st.prepare_grow(512, (0, 1)) > 0
    st.resize(32)                       # adopts the prepared tail, then retires it
    assert st.read_cell("a", 0, 299, 1) == keep
    st.reclaim()
    assert st.vmm_stats()["pending_reclaim_bytes"] == 0
    st.resize(128)
    st.append_seeded("b", 1, 16 * 100, 2)
    for _ in range(3):
        t = kv.KvStore(1, 2, 16, 64, (0,), cell_bytes=4096, chunk_bytes=2 << 20)
        t.prepare_grow(1024, (0,))
        del t                           # prepared tail never adopted


def test_acceptance_criterion_3_randomized_allocator_ops():
    """Acceptance criterion 3 (pkg/tests/test_acceptance.py:104-150): 10,500 randomized
    append / free / compact / resize ops on a 48-block store (k=2, 8-token blocks, two
    groups) never lose a checksum, shrink-below-live fires exactly when live > target,
    within 10 s -- here on the GPU store, checked against a host shadow."""
    import random
    import time

    from paper_2604_12171_b200 import kvstore as kv

    t0 = time.time()
    rng = random.Random(3003)
    st = kv.KvStore(1, 2, 8, 48, (0, 1))
    shadow: dict = {}
    reqs = [f"r{i}" for i in range(10)]
    for op in range(1, 10_501):
        roll, req = rng.random(), rng.choice(reqs)
        if roll < 0.5:
            g, n = rng.choice((0, 1)), rng.randint(1, 20)
            pay = [rng.randrange(2 ** 40) for _ in range(n)]
            try:
                st.append(req, g, n, pay)
                shadow.setdefault((req, g), []).extend(pay)
            except kv.KvOverflow:
                pass
        elif roll < 0.65:
            st.free_request(req)
            shadow.pop((req, 0), None)
            shadow.pop((req, 1), None)
        elif roll < 0.8:
            st.compact()
        else:
            target, live = rng.randint(0, 56), st.used_blocks
            try:
                st.resize(target)
                assert live <= target
            except kv.CapacityBelowLive:
                assert live > target
        if op % 500 == 0:
            for (rid, g), pays in shadow.items():
                for pos in range(len(pays)):
                    assert st.read_checksum(rid, g, pos) == pays[pos]
        else:
            for (rid, g), pays in list(shadow.items())[:3]:
                pos = rng.randrange(len(pays))
                assert st.read_checksum(rid, g, pos) == pays[pos]
    assert time.time() - t0 < 10.0, time.time() - t0


class TestLazyGroupAdoption:
    """A group added while the reclaimer thread is busy is mapped lazily; the first
    allocation must adopt it over the whole capacity (ensure_slots used to
    clear the pending bit and map only up to the allocated slot, while chains shared
    with other groups already held live blocks at higher slots)."""

    def test_new_group_written_at_high_slots_while_reclaimer_busy(self, kv):
        import ctypes as C

        import torch

        from paper_2604_12171_b200 import _native as N

        st = kv.KvStore(1, 2, 16, 64, (0, 1), cell_bytes=4096, chunk_bytes=2 << 20)
        s = torch.cuda.Stream()
        N.check(N.lib().pl_store_set_stream(st._h, C.c_void_p(s.cuda_stream)))
        for i in range(60):
            st.append_seeded(f"x{i}", 0, 16, 100 + i)
        for i in range(0, 40):
            st.free_request(f"x{i}")          # holes in the low slots, live blocks above
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000_000)    # ~0.1 s: the release job below waits on it
        st.drop_layer_groups([1])             # immediate reclaim job, gated on the sleep
        st.resident_groups.add(2)             # lazy pool: its mapping queues behind the job
        st.append_seeded("new", 2, 16, 7)     # allocates a low hole first
        for i in range(40, 60):               # then the shared chains at high slots
            st.append_seeded(f"x{i}", 2, 16, 200 + i)
        st.sync()
        for i in range(40, 60):
            fp = st.read_checksum(f"x{i}", 2, 15)
            assert st.read_cell(f"x{i}", 2, 15, 1) == oracle.expand_cell(fp, 1, 4096)
        # a shrink relocates the live high units of every group, the new one included
        keep = {(f"x{i}", g): st.read_cell(f"x{i}", g, 3, 0) for i in range(40, 60) for g in (0, 2)}
        st.compact()
        st.resize(st.used_blocks + 1)
        assert st.last_resize_stats()["relocated_blocks"] > 0
        for (r, g), v in keep.items():
            assert st.read_cell(r, g, 3, 0) == v
        torch.cuda.synchronize()


def test_upload_ring_outgrows_without_a_host_sync_and_frees_at_sync():
    """Uploads larger than a quarter of the H2D staging ring take a larger ring; the
    outgrown ones are freed at the next sync() (a host sync point), not inside an upload
    (cudaFree / cudaFreeHost would stall the device queue there), and every payload
    staged through the old and new rings lands in its cells."""
    from paper_2604_12171_b200 import kvstore as kv
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import append_batch_payloads, engine_payloads

    reg = kv.RequestRegistry()
    st = kv.KvStore(1, 2, 16, 16384, (0, 1), cell_bytes=64, registry=reg)
    s0 = st.staging_stats()
    seeds = {}
    for j, (n_req, n_tok) in enumerate(((16, 512), (64, 512), (64, 1024))):
        names = [f"u{j}_{i}" for i in range(n_req)]
        reqs = [reg.handle(r) for r in names for _ in (0, 1)]
        groups = [g for _ in names for g in (0, 1)]
        pls = []
        for r in names:
            for g in (0, 1):
                seeds[(r, g)] = stable_hash(r, g)
                pls.append(engine_payloads(seeds[(r, g)], n_tok))
        assert append_batch_payloads(st, reqs, groups, [n_tok] * len(reqs),
                                     np.concatenate(pls)) == len(reqs)
    s1 = st.staging_stats()
    assert s1["outgrows"] - s0["outgrows"] >= 2 and s1["old_rings"] >= 1, (s0, s1)
    st.sync()
    assert st.staging_stats()["old_rings"] == 0
    out = st.verify_cells(seeds)
    assert out["cells"] > 0 and out["bad_bytes"] == 0 and out["bad_fingerprints"] == 0, out


def test_large_payload_upload_is_copied_exactly():
    """A bulk append's payload upload (8 MB here, configs[1]'s shape: 256 requests x 2
    groups x 2048 tokens) is copied into the pinned staging ring by several threads
    (store.cu copy_part); every fingerprint must land in its cell."""
    from paper_2604_12171_b200 import kvstore as kv
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import append_batch_payloads, engine_payloads

    reg = kv.RequestRegistry()
    st = kv.KvStore(1, 2, 16, 33000, (0, 1), cell_bytes=64, registry=reg)
    names = [f"big{i}" for i in range(256)]
    reqs = [reg.handle(r) for r in names for _ in (0, 1)]
    groups = [g for _ in names for g in (0, 1)]
    seeds = {(r, g): stable_hash(r, g) for r in names for g in (0, 1)}
    pls = np.concatenate([engine_payloads(seeds[(r, g)], 2048) for r in names for g in (0, 1)])
    assert pls.nbytes >= 8 << 20
    assert append_batch_payloads(st, reqs, groups, [2048] * len(reqs), pls) == len(reqs)
    st.sync()
    out = st.verify_cells(seeds)
    assert out["cells"] == 256 * 2 * 2048, out   # (position, group) pairs, k layers each
    assert out["bad_bytes"] == 0 and out["bad_fingerprints"] == 0, out
