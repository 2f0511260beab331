"""GPU KV-patching parity: dirty sets, patch counters, traces and patched bytes of
the CUDA patch engine against the reference (tests/golden/migration_cases.json)
and the oracle.  Mirrors pkg/tests/test_migrator.py of the reference."""

import ctypes as C

import numpy as np
import pytest

import opgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ns():
    from paper_2604_12171_b200 import events, fabric, kvstore, migrator

    class NS:
        EventScheduler = events.EventScheduler
        EventTrace = events.EventTrace
        CommFabric = fabric.CommFabric
        FabricConfig = fabric.FabricConfig
        KvStore = kvstore.KvStore
        MigrationManager = migrator.MigrationManager

    return NS


@pytest.fixture
def drain_log(monkeypatch):
    """Record the drained key set of every patch, and check the device's view of it."""
    from paper_2604_12171_b200 import migrator

    log = []
    orig = migrator.MigrationStream._drain

    def drain(self):
        host_dirty = self._dirty_keys()
        dev_dirty = self.device_dirty_count()
        assert dev_dirty == host_dirty, "device bitmap != host dirty set"
        patch = orig(self)
        keys = self.drained_keys()
        assert self.device_drained() == len(keys) == patch.keys
        log.append([list(k) for k in keys])
        return patch

    monkeypatch.setattr(migrator.MigrationStream, "_drain", drain)
    return log


@pytest.mark.parametrize("seed", range(80))
def test_gpu_migration_matches_reference(ns, golden, drain_log, seed):
    case = golden("migration_cases.json")[seed]
    res = opgen.run_migration_case(ns, case["case"], {"cell_bytes": 64})
    want = dict(case["result"])
    assert drain_log == want.pop("drained")  # dirty sets, patch by patch
    assert res == want


def test_patched_bytes_are_bit_exact(ns, drain_log):
    """Destination KV bytes == source bytes == expansion of the reference fingerprint."""
    from paper_2604_12171_b200 import kvstore

    case = opgen.migration_case(3)
    case["events"] = []
    cb = 4096
    sched = ns.EventScheduler()
    trace = ns.EventTrace()
    fab = ns.CommFabric(sched, trace, [1, 2], ns.FabricConfig())
    k, s = 4, 16
    src = kvstore.KvStore(1, k, s, 64, [0, 1, 2], cell_bytes=cb)
    dst = kvstore.KvStore(2, k, s, 64, [5], cell_bytes=cb)
    mgr = ns.MigrationManager(sched, trace, fab, {1: src, 2: dst}, 8192, k)
    for i in range(6):
        for g in (0, 1, 2):
            n = 7 + 13 * i
            src.append(f"b{i}", g, n, [opgen.payload(f"b{i}", g, p) for p in range(n)])
    dst.resident_groups |= {1, 2}
    mgr.start_migration({(1, 2): set(range(5, 13))})
    sched.run()
    assert mgr.lag(2) == 0
    for g in (1, 2):
        assert dst.snapshot_group(g) == src.snapshot_group(g)
        for rid, fps in src.snapshot_group(g).items():
            for pos in (0, len(fps) // 2, len(fps) - 1):
                for j in range(k):
                    b = dst.read_cell(rid, g, pos, j)
                    assert b == src.read_cell(rid, g, pos, j)
                    assert b == oracle.expand_cell(fps[pos], j, cb)


def test_stacked_groups_count_cells_not_tokens(ns):
    from paper_2604_12171_b200 import kvstore

    sched, trace = ns.EventScheduler(), ns.EventTrace()
    fab = ns.CommFabric(sched, trace, [1, 2], ns.FabricConfig())
    src = kvstore.KvStore(1, 4, 16, 64, (0, 1))
    dst = kvstore.KvStore(2, 4, 16, 64, (2,))
    mgr = ns.MigrationManager(sched, trace, fab, {1: src, 2: dst}, 8192, 4)
    src.append("a", 0, 10, [opgen.payload("a", 0, p) for p in range(10)])
    mgr.start_migration({(1, 2): {1, 2, 3, 4}})
    assert mgr.counters.t_sched[2] == 40
    sched.run()
    assert mgr.lag(2) == 0


def test_final_sync_residual_arithmetic(ns):
    from paper_2604_12171_b200 import kvstore

    sched, trace = ns.EventScheduler(), ns.EventTrace()
    fab = ns.CommFabric(sched, trace, [1, 2], ns.FabricConfig())
    src = kvstore.KvStore(1, 1, 16, 64, (0, 1))
    dst = kvstore.KvStore(2, 1, 16, 64, (2,))
    mgr = ns.MigrationManager(sched, trace, fab, {1: src, 2: dst}, 8192, 1)
    mgr.start_migration({(1, 2): {1}})
    sched.run()
    mgr.streams[(1, 2)].streaming = False
    src.append("a", 0, 40, [opgen.payload("a", 0, p) for p in range(40)])
    mgr.on_kv_written(1, "a", 0, 0, 40)
    pauses = []
    mgr.final_sync_all(pauses.append)
    sched.run()
    transfer = 40 * 8192 / fab.bandwidth(1, 2)
    assert transfer == pytest.approx(2.62144e-05)
    assert pauses[0] == pytest.approx(transfer + 2e-4)
    assert dst.snapshot_group(0) == src.snapshot_group(0)


def test_push_path_direct_into_destination(ns):
    """perf path: drain + fused gather/scatter straight into the destination pool"""
    import ctypes as C

    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200 import kvstore

    src = kvstore.KvStore(1, 2, 16, 128, (0, 1), cell_bytes=1024)
    dst = kvstore.KvStore(2, 2, 16, 128, (3,), cell_bytes=1024)
    for i in range(10):
        src.append_seeded(f"p{i}", 1, 30 + i, opgen.stable_hash(f"p{i}", 1))
    dst.resident_groups |= {1}
    g = N.as_i32([1])
    lpg = N.as_i32([2])
    h = C.c_void_p()
    N.check(N.lib().pl_patch_create(src._h, N.ptr(g), N.ptr(lpg), 1, C.byref(h)))
    N.check(N.lib().pl_patch_set_active(h, 1))
    seeded = C.c_int64()
    N.check(N.lib().pl_patch_seed(h, C.byref(seeded)))
    rank = src._registry.rank()
    keys, cells = C.c_int64(), C.c_int64()
    N.check(N.lib().pl_patch_push(h, dst._h, N.ptr(rank), len(rank), C.byref(keys), C.byref(cells)))
    assert keys.value == seeded.value == sum(30 + i for i in range(10))
    assert cells.value == 2 * keys.value
    assert dst.snapshot_group(1) == src.snapshot_group(1)
    for i in range(10):
        assert dst.read_cell(f"p{i}", 1, 29 + i, 1) == src.read_cell(f"p{i}", 1, 29 + i, 1)
    N.lib().pl_patch_destroy(h)


@pytest.mark.parametrize("seed,chunked", [(0, False), (1, False), (2, False), (0, True), (3, True)])
def test_side_stream_push_overlapped_with_decode_writes(monkeypatch, seed, chunked):
    """K3/K4/K5 on a low-priority side stream while K1 keeps writing (and marking) on the
    store's stream with no host sync in between: after the final round the destination
    holds exactly the source's migrating groups, byte for byte, and requests freed
    mid-migration are gone from both.  `chunked`: every round that allocates destination
    blocks takes the pipelined multi-launch path."""
    if chunked:
        monkeypatch.setenv("PL_PUSH_CHUNK_MIN_BLOCKS", "1")
        monkeypatch.setenv("PL_PUSH_CHUNK_ALWAYS", "1")
    import random

    import torch

    from paper_2604_12171_b200 import kvstore
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import NativePatch

    rng = random.Random(seed)
    reg = kvstore.RequestRegistry()
    names = [f"q{i:03d}" for i in range(40)]
    for n in names:
        reg.handle(n)
    src = kvstore.KvStore(1, 2, 16, 2048, (0, 1, 2), num_groups=3, cell_bytes=512, registry=reg)
    dst = kvstore.KvStore(2, 2, 16, 2048, (), num_groups=3, cell_bytes=512, registry=reg)
    dst.resident_groups |= {1, 2}
    lo, _ = torch.cuda.Stream.priority_range()
    side = torch.cuda.Stream(priority=lo)
    for n in names[:30]:
        for g in range(3):
            src.append_seeded(n, g, 1 + rng.randrange(200), stable_hash(n, g))
    p = NativePatch(src, (1, 2), 2)
    p.set_stream(side.cuda_stream)
    p.seed()
    p.push(dst, reg.rank())                    # bulk, no sync afterwards
    live = set(names[:30])
    for step in range(25):
        for n in rng.sample(sorted(live | set(names[30:])), 12):
            for g in range(3):
                src.append_seeded(n, g, 1 + rng.randrange(5), stable_hash(n, g), mark=True)
            live.add(n)
        if step % 7 == 3:                      # a request finishes mid-migration
            gone = rng.choice(sorted(live))
            live.discard(gone)
            p.discard_request(gone, reg)
            src.free_request(gone)
            dst.free_request(gone)
        p.push(dst, reg.rank())                # one round per step, no host sync
    p.push(dst, reg.rank())                    # residual
    torch.cuda.synchronize()
    for g in (1, 2):
        assert dst.snapshot_group(g) == src.snapshot_group(g)
        for rid, fps in src.snapshot_group(g).items():
            for pos in {0, len(fps) // 2, len(fps) - 1}:
                assert dst.read_cell(rid, g, pos, 1) == src.read_cell(rid, g, pos, 1)
    assert p.dirty_keys() == 0
    p.close()


def _chunk_rig(cap_dst, n_req=48, seed=0):
    import random

    from paper_2604_12171_b200 import kvstore
    from paper_2604_12171_b200.events import stable_hash

    rng = random.Random(seed)
    reg = kvstore.RequestRegistry()
    names = [f"c{i:03d}" for i in range(n_req)]
    for n in names:
        reg.handle(n)
    src = kvstore.KvStore(1, 2, 16, 4096, (0, 1, 2), num_groups=3, cell_bytes=256, registry=reg)
    dst = kvstore.KvStore(2, 2, 16, cap_dst, (), num_groups=3, cell_bytes=256, registry=reg)
    dst.resident_groups |= {1, 2}
    for n in names:
        for g in range(3):
            src.append_seeded(n, g, 1 + rng.randrange(300), stable_hash(n, g))
    return reg, names, src, dst


def _dst_state(dst, names):
    tables = {n: [b.block_id for b in dst.tables[n].chain] for n in names if n in dst.tables}
    cells = {(n, g, p): dst.read_cell(n, g, p, j)
             for n in names if n in dst.tables for g in (1, 2)
             for p in {0, dst.tables[n].written.get(g, 1) - 1} if dst.tables[n].written.get(g, 0)
             for j in (0, 1)}
    return tables, {g: dst.snapshot_group(g) for g in (1, 2)}, cells, dst.used_blocks


@pytest.mark.parametrize("cap_dst,seed", [(4096, 0), (4096, 1), (300, 2)])
def test_chunked_bulk_push_equals_single_launch(monkeypatch, cap_dst, seed):
    """A cold bulk round that allocates many destination blocks is reserved and copied in
    pipelined runs (Patch::push_chunked).  Forced down to tiny runs, it must leave the
    destination exactly as the one-launch push does: same block ids (allocation order),
    same fingerprints and bytes -- and, when the destination overflows mid-round, the
    same applied prefix and the same KvOverflow."""
    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200.perf import NativePatch

    states = []
    for chunked in (False, True):
        if chunked:
            monkeypatch.delenv("PL_PUSH_NO_CHUNK", raising=False)
            monkeypatch.setenv("PL_PUSH_CHUNK_MIN_BLOCKS", "1")
            monkeypatch.setenv("PL_PUSH_CHUNK_ALWAYS", "1")
        else:
            monkeypatch.setenv("PL_PUSH_NO_CHUNK", "1")
        reg, names, src, dst = _chunk_rig(cap_dst, seed=seed)
        p = NativePatch(src, (1, 2), 2)
        p.seed()
        N.check(N.lib().pl_timing_reset())
        N.check(N.lib().pl_timing_enable(1))
        overflow = None
        try:
            p.push(dst, reg.rank())
        except N.NativeError as e:
            assert e.code == -1            # PL_E_KV_OVERFLOW -> KvOverflow
            overflow = str(e)
        src.sync()
        dst.sync()
        launches = N.timing("patch_push")[1]
        N.check(N.lib().pl_timing_enable(0))
        states.append((overflow, _dst_state(dst, names)))
        if chunked:
            assert launches > 2, launches
        else:
            assert launches == 1
        if cap_dst >= 4096:
            assert overflow is None
            for g in (1, 2):
                assert dst.snapshot_group(g) == src.snapshot_group(g)
        else:
            assert overflow is not None
        p.close()
        src.close()
        dst.close()
    assert states[0] == states[1]


def test_cold_round_pipelines_only_when_the_device_waits(monkeypatch):
    """A cold round pipelines its host reservation with the copy (Patch::push_chunked)
    unless the caller already runs ahead of the device: with milliseconds of work queued
    on the source's stream the reservation is hidden behind it, and the round goes out as
    one launch (Patch::runs_ahead).  Either way the destination is the same."""
    import torch

    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200.perf import NativePatch

    monkeypatch.setenv("PL_PUSH_CHUNK_MIN_BLOCKS", "1")
    monkeypatch.delenv("PL_PUSH_CHUNK_ALWAYS", raising=False)
    monkeypatch.delenv("PL_PUSH_NO_CHUNK", raising=False)
    states = []
    for busy in (False, True):
        reg, names, src, dst = _chunk_rig(4096, seed=3)
        p = NativePatch(src, (1, 2), 2)
        p.seed()
        src.sync()
        if busy:   # ~20 ms of queued work on the source's stream (a caller running ahead)
            out = C.c_void_p()
            N.check(N.lib().pl_store_stream(src._h, C.byref(out)))
            with torch.cuda.stream(torch.cuda.ExternalStream(out.value)):
                torch.cuda._sleep(40_000_000)
        N.check(N.lib().pl_timing_reset())
        N.check(N.lib().pl_timing_enable(1))
        p.push(dst, reg.rank())
        stats = p.last_push_stats()
        src.sync()
        dst.sync()
        launches = N.timing("patch_push")[1]
        N.check(N.lib().pl_timing_enable(0))
        assert stats["chunked"] is (not busy), stats
        assert (launches == 1) if busy else (launches > 2), launches
        states.append(_dst_state(dst, names))
        p.close()
        src.close()
        dst.close()
    assert states[0] == states[1]


def test_concurrent_pairs_on_separate_streams():
    """configs[4]'s pairs axis, for correctness: several independent (src, dst) pairs push
    on their own low-priority streams with no host sync between them -- cold bulk rounds
    (pipelined runs) and a steady round after new writes -- and every destination ends up
    equal to its source, fingerprints and sampled bytes."""
    import random

    import torch

    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.perf import PatchRig, Workload, append_batch, rid

    wl = Workload(batch=24, ctx=300)
    lo, _ = torch.cuda.Stream.priority_range()
    rigs = []
    for _ in range(4):
        rig = PatchRig(wl)
        rig.fill()
        s = torch.cuda.Stream(priority=lo)
        rig.patch.set_stream(s.cuda_stream)
        rigs.append((rig, s))
    for rig, _ in rigs:
        rig.patch.seed()
    for rig, _ in rigs:                               # cold bulk rounds, all in flight
        rig.patch.push(rig.dst, rig.registry.rank())
    for n, (rig, _) in enumerate(rigs):               # new tokens while the copies run
        append_batch(rig.src, rig.handles, [wl.mig_groups[0]] * wl.batch, [3] * wl.batch,
                     [stable_hash(rid(i), wl.mig_groups[0]) for i in range(wl.batch)], mark=True)
    for rig, _ in rigs:
        rig.patch.push(rig.dst, rig.registry.rank())
    torch.cuda.synchronize()
    rng = random.Random(3)
    for rig, _ in rigs:
        for g in wl.mig_groups:
            assert rig.dst.snapshot_group(g) == rig.src.snapshot_group(g)
            for _ in range(6):
                i = rng.randrange(wl.batch)
                pos = rng.randrange(wl.ctx + (3 if g == wl.mig_groups[0] else 0))
                assert rig.dst.read_cell(rid(i), g, pos, 1) == rig.src.read_cell(rid(i), g, pos, 1)
        rig.destroy()


@pytest.mark.parametrize("side_stream", [False, True])
def test_perf_push_edge_rounds(side_stream):
    """The perf push (pl_patch_push) through the round shapes a live migration meets, each
    checked byte for byte against the source (every written position, fingerprint + k
    cells, through both block tables): ragged request lengths (1 .. 2 blocks + 1) in the
    bulk round; an empty round; a launch-first steady round (every position inside an
    existing destination block); a round that needs new destination blocks; a round in
    which a request finished after its writes were marked (discarded, not shipped)."""
    import torch

    from paper_2604_12171_b200 import kvstore
    from paper_2604_12171_b200.perf import NativePatch, append_batch

    reg = kvstore.RequestRegistry()
    k, s = 2, 16
    src = kvstore.KvStore(1, k, s, 512, (0, 1, 2), num_groups=3, cell_bytes=4096, registry=reg)
    dst = kvstore.KvStore(2, k, s, 512, (2,), num_groups=3, cell_bytes=4096, registry=reg)
    dst.resident_groups |= {0, 1}
    lens = [1, 15, 16, 17, 31, 32, 33, 5]
    names = [f"e{i}" for i in range(len(lens))]
    hs = [reg.handle(n) for n in names]
    seeds = {(n, g): opgen.stable_hash(n, g) for n in names for g in (0, 1, 2)}

    def append(which, counts, mark):
        reqs = [hs[i] for i in which for _ in (0, 1, 2)]
        groups = [g for _ in which for g in (0, 1, 2)]
        cnt = [counts[i] for i in which for _ in (0, 1, 2)]
        sd = [seeds[(names[i], g)] for i in which for g in (0, 1, 2)]
        assert append_batch(src, reqs, groups, cnt, sd, mark=mark) == len(reqs)

    def same(live):
        src.sync()
        dst.sync()
        out = src.compare_cells(dst, (0, 1), [names[i] for i in live])
        assert out["bad_positions"] == 0 and out["missing"] == 0, out
        assert out["length_mismatch"] == 0, out
        return out["cells"]

    append(range(len(lens)), lens, mark=False)
    patch = NativePatch(src, (0, 1), k)
    side = torch.cuda.Stream() if side_stream else None
    if side is not None:
        patch.set_stream(side.cuda_stream)
    assert patch.seed() == 2 * sum(lens)
    keys, cells = patch.push(dst, reg.rank())
    assert (keys, cells) == (2 * sum(lens), 2 * k * sum(lens))
    assert same(range(len(lens))) == 2 * sum(lens) * k
    # empty round
    assert patch.push(dst, reg.rank()) == (0, 0)
    assert patch.device_drained() == 0
    # steady decode round: one token per request, group 2 (not migrating) too; positions
    # 2..16 -> 15, 16, 17 ... lie inside existing destination blocks except lens 16 / 32
    inside = [i for i, n in enumerate(lens) if n % s != 0]
    append(inside, [1] * len(lens), mark=True)
    keys, _ = patch.push(dst, reg.rank())
    assert keys == 2 * len(inside) and patch.device_drained() == keys
    lens = [n + 1 if i in inside else n for i, n in enumerate(lens)]
    same(range(len(lens)))
    # a round whose positions need new destination blocks (16 -> 17, 32 -> 33 and more)
    append(range(len(lens)), [s] * len(lens), mark=True)
    keys, _ = patch.push(dst, reg.rank())
    assert keys == 2 * s * len(lens)
    lens = [n + s for n in lens]
    same(range(len(lens)))
    # a request finishes after its writes were marked: discarded, never shipped
    append(range(len(lens)), [3] * len(lens), mark=True)
    gone = 3
    assert patch.discard_request(names[gone], reg) > 0
    src.free_request(names[gone])
    dst.free_request(names[gone])
    keys, _ = patch.push(dst, reg.rank())
    assert keys == 2 * 3 * (len(lens) - 1)
    lens = [n + 3 for n in lens]
    live = [i for i in range(len(lens)) if i != gone]
    same(live)
    patch.close()
