"""The reference's KV-store test suite (pkg/tests/test_kvstore.py), restated against the
GPU-backed drop-in.  Same test names and the same asserted behaviour, so a reader can
put the two files side by side; every store here keeps its blocks in VMM pools on the
device and every append runs K1.  Builders mirror pkg/tests/helpers.py:13-33."""

import random

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

KIB, MIB = 1024, 1024 * 1024


def _ps():
    import paper_2604_12171_b200 as ps
    from paper_2604_12171_b200 import kvstore
    return ps, kvstore


def gpu_spec(mem_mib=4096, gran_mib=2):
    ps, _ = _ps()
    return ps.GpuSpec(1, mem_mib * MIB, 1e12, 1e-5, 1e-5, gran_mib * MIB)


def model_spec(layers=8, k=1, weight_mib=64, token_kv=8 * KIB):
    ps, _ = _ps()
    return ps.ModelSpec(layers, weight_mib * MIB, token_kv, k)


def store_of(capacity=10, s=16, k=4, groups=(0,)):
    _, kv = _ps()
    return kv.KvStore(gpu_id=1, stacking_factor=k, tokens_per_block=s,
                      capacity_blocks=capacity, resident_groups=groups)


def fp(req, group, pos):
    from paper_2604_12171_b200.events import stable_hash
    return stable_hash(req, group, pos)


def put(store, req, group, n):
    """Append n tokens continuing the request's group, payload = stable_hash fingerprints."""
    start = store.tables[req].written.get(group, 0) if req in store.tables else 0
    return store.append(req, group, n, [fp(req, group, start + i) for i in range(n)])


# --- TestInit (test_kvstore.py:40-60) ------------------------------------------------------
def test_zero_capacity_store_is_valid():
    _, kv = _ps()
    st_ = kv.kv_init(gpu_spec(), model_spec(), 0)
    assert st_.capacity_blocks == 0
    with pytest.raises(kv.KvOverflow):
        st_.append("r1", 0, 1, [1])


def test_tokens_per_block_geometry():
    _, kv = _ps()
    # 2 MiB granule / (8 KiB per token-layer x k = 4) = 64 tokens per block
    st_ = kv.kv_init(gpu_spec(gran_mib=2), model_spec(layers=8, k=4), 10, resident_groups=(0, 1))
    assert st_.tokens_per_block == 64


def test_capacity_exceeding_memory_rejected():
    _, kv = _ps()
    with pytest.raises(kv.InsufficientMemory):
        kv.kv_init(gpu_spec(mem_mib=64), model_spec(layers=4, k=1), 1000,
                   resident_groups=range(4))


# --- TestAppend (test_kvstore.py:63-102) ---------------------------------------------------
def test_append_zero_tokens():
    st_ = store_of()
    assert st_.append("r1", 0, 0, []) == []
    assert st_.used_blocks == 0


def test_fresh_request_40_tokens_three_blocks():
    st_ = store_of(s=16)
    slots = put(st_, "r1", 0, 40)
    assert st_.used_blocks == 3
    assert [x.offset for x in slots] == [*range(16), *range(16), *range(8)]
    assert [x.block_id for x in slots] == [0] * 16 + [1] * 16 + [2] * 8


def test_overflow_when_full():
    _, kv = _ps()
    st_ = store_of(capacity=2, s=16)
    put(st_, "r1", 0, 32)
    with pytest.raises(kv.KvOverflow):
        put(st_, "r1", 0, 1)


def test_overflow_is_atomic():
    _, kv = _ps()
    st_ = store_of(capacity=2, s=16)
    put(st_, "r1", 0, 20)
    with pytest.raises(kv.KvOverflow):
        put(st_, "r2", 0, 40)
    assert st_.used_blocks == 2 and "r2" not in st_.tables


def test_chain_shared_across_groups():
    st_ = store_of(capacity=4, s=16, groups=(0, 1))
    put(st_, "r1", 0, 20)
    put(st_, "r1", 1, 20)
    assert st_.used_blocks == 2     # one chain, both groups stacked in its two blocks


# --- TestLookup (test_kvstore.py:105-126) --------------------------------------------------
@pytest.mark.parametrize("n,tok,entry,off", [(5, 0, 0, 0), (25, 20, 1, 4)],
                         ids=["test_first_token", "test_token_20_resolves_to_second_entry"])
def test_lookup_resolves_through_chain(n, tok, entry, off):
    st_ = store_of(s=16)
    put(st_, "r1", 0, n)
    assert st_.lookup("r1", 1, tok) == (st_.tables["r1"].chain[entry].address, off)


def test_unknown_beyond_range():
    _, kv = _ps()
    st_ = store_of(s=16)
    put(st_, "r1", 0, 5)
    for req, tok in (("r1", 5), ("r2", 0)):
        with pytest.raises(kv.UnknownSlot):
            st_.lookup(req, 1, tok)


# --- TestCompact (test_kvstore.py:129-165) -------------------------------------------------
def _fragmented():
    st_ = store_of(capacity=5, s=16)
    for req in "abcde":
        put(st_, req, 0, 16)
    st_.free_request("b")
    st_.free_request("d")
    return st_   # block order = allocation order: a, b(free), c, d(free), e


def test_live_free_partition():
    st_ = _fragmented()
    assert [b.state for b in st_.blocks] == ["live", "free", "live", "free", "live"]
    assert st_.compact() == 2
    assert [b.state for b in st_.blocks] == ["live"] * 3 + ["free"] * 2


@pytest.mark.parametrize("fill", [True, False],
                         ids=["test_no_free_blocks_is_noop", "test_all_free_preserves_order"])
def test_compact_keeps_order_when_nothing_interleaves(fill):
    st_ = store_of(capacity=2 if fill else 4, s=16)
    if fill:
        put(st_, "a", 0, 32)
    ids = [b.block_id for b in st_.blocks]
    assert st_.compact() == (0 if fill else 4)
    assert [b.block_id for b in st_.blocks] == ids


def test_lookups_and_checksums_survive():
    st_ = _fragmented()
    want = {(r, p): st_.lookup(r, 1, p) for r in "ace" for p in range(16)}
    st_.compact()
    for (r, p), addr in want.items():
        assert st_.lookup(r, 1, p) == addr
        assert st_.read_checksum(r, 0, p) == fp(r, 0, p)


# --- TestResize (test_kvstore.py:168-210) --------------------------------------------------
def test_shrink_after_compaction():
    st_ = store_of(capacity=10, s=16)
    for req in "abcd":
        put(st_, req, 0, 16)
    st_.compact()
    st_.resize(6)
    assert (st_.capacity_blocks, st_.used_blocks) == (6, 4)


def test_shrink_below_live_rejected():
    _, kv = _ps()
    st_ = store_of(capacity=10, s=16)
    for req in "abcdefg":
        put(st_, req, 0, 16)
    with pytest.raises(kv.CapacityBelowLive):
        st_.resize(6)
    assert st_.capacity_blocks == 10


def test_resize_to_current_is_noop():
    st_ = store_of(capacity=10)
    ids = [b.block_id for b in st_.blocks]
    st_.resize(10)
    assert [b.block_id for b in st_.blocks] == ids


def test_round_trip_restores_capacity_and_lookups():
    st_ = store_of(capacity=10, s=16)
    put(st_, "a", 0, 40)
    addrs = [st_.lookup("a", 1, i) for i in range(40)]
    st_.resize(5)
    st_.resize(10)
    assert st_.capacity_blocks == 10
    assert [st_.lookup("a", 1, i) for i in range(40)] == addrs


def test_expand_adds_free_blocks():
    st_ = store_of(capacity=2, s=16)
    put(st_, "a", 0, 32)
    st_.resize(4)
    put(st_, "a", 0, 32)
    assert st_.used_blocks == 4


# --- TestDropLayers (test_kvstore.py:213-246) ----------------------------------------------
def test_drop_all_groups_zeroes_usage():
    st_ = store_of(capacity=8, s=16, groups=(0, 1))
    put(st_, "a", 0, 16)
    put(st_, "a", 1, 16)
    assert st_.drop_layer_groups([0, 1]) == 32
    assert st_.used_blocks == 0


def test_drop_one_group_keeps_shared_blocks_live():
    st_ = store_of(capacity=8, s=16, groups=(0, 1))
    put(st_, "a", 0, 32)
    put(st_, "a", 1, 32)
    assert st_.used_blocks == 2
    occ = sum(b.occupied_tokens() for b in st_.blocks)
    assert st_.drop_layer_groups([0]) == 32
    assert st_.used_blocks == 2                       # group 1 still lives in both blocks
    assert st_.read_checksum("a", 1, 17) == fp("a", 1, 17)
    assert sum(b.occupied_tokens() for b in st_.blocks) == occ // 2


def test_drop_empty_group():
    st_ = store_of(groups=(0, 1))
    put(st_, "a", 0, 4)
    assert st_.drop_layer_groups([1]) == 0


def test_unknown_group_rejected():
    _, kv = _ps()
    with pytest.raises(kv.UnknownLayerGroup):
        store_of(groups=(0,)).drop_layer_groups([3])


# --- TestUtilization / TestStackingConservation (test_kvstore.py:249-295) ------------------
@pytest.mark.parametrize("s,n,want", [(16, 64, 1.0), (64, 16, 0.25), (16, 0, 1.0)],
                         ids=["test_full_blocks_are_1", "test_quarter_filled_block",
                              "test_idle_store_is_vacuously_1"])
def test_effective_utilization(s, n, want):
    st_ = store_of(capacity=4, s=s, groups=(0,))
    if n:
        put(st_, "a", 0, n)
    assert st_.effective_utilization() == want


def test_stacking_beats_unstacked_on_short_requests():
    _, kv = _ps()
    util = {}
    for k in (1, 4):
        groups = range(4 // k)
        st_ = kv.kv_init(gpu_spec(), model_spec(layers=4, k=k), 64, resident_groups=groups)
        n = st_.tokens_per_block // 4 + 1          # straddles a block edge
        for g in groups:
            for req in "abc":
                st_.append(req, g, n, [fp(req, g, i) for i in range(n)])
        util[k] = st_.effective_utilization()
    assert util[4] > util[1]


def test_total_cell_capacity_independent_of_k():
    _, kv = _ps()
    cells = {(lambda st_: st_.capacity_blocks * st_.tokens_per_block * k)(
        kv.kv_init(gpu_spec(), model_spec(layers=8, k=k), 32, resident_groups=range(8 // k)))
        for k in (1, 2, 4, 8)}
    assert len(cells) == 1


@given(st.integers(1, 200), st.sampled_from([4, 8, 16, 64]))
@settings(max_examples=40, deadline=None)
def test_fragmentation_bound_exact(req_tokens, s):
    _, kv = _ps()
    st_ = kv.KvStore(gpu_id=1, stacking_factor=1, tokens_per_block=s, capacity_blocks=64,
                     resident_groups=(0,))
    put(st_, "r", 0, req_tokens)
    u = st_.effective_utilization()
    assert u == req_tokens / (-(-req_tokens // s) * s)
    assert u >= req_tokens / (req_tokens + s - 1)


@given(st.integers(0, 2 ** 32 - 1))
@settings(max_examples=12, deadline=None)
def test_randomized_ops_preserve_shadow_model(seed):
    """append / free / compact / resize fuzz against a dict shadow of every payload."""
    _, kv = _ps()
    rng = random.Random(seed)
    s = rng.choice([4, 8, 16])
    st_ = kv.KvStore(1, 2, s, capacity_blocks=24, resident_groups=(0, 1))
    shadow = {}
    reqs = [f"r{i}" for i in range(6)]
    for _ in range(120):
        x, req = rng.random(), rng.choice(reqs)
        if x < 0.55:
            g = rng.choice((0, 1))
            n = rng.randint(1, 2 * s)
            base = len(shadow.get((req, g), []))
            pay = [fp(req, g, base + i) for i in range(n)]
            try:
                st_.append(req, g, n, pay)
            except kv.KvOverflow:
                continue
            shadow.setdefault((req, g), []).extend(pay)
        elif x < 0.7:
            st_.free_request(req)
            shadow.pop((req, 0), None)
            shadow.pop((req, 1), None)
        elif x < 0.85:
            st_.compact()
        else:
            b = rng.randint(0, 30)
            try:
                st_.resize(b)
            except kv.CapacityBelowLive:
                assert st_.used_blocks > b
        for (r, g), pay in shadow.items():
            for p in (0, len(pay) - 1, rng.randrange(len(pay))):
                assert st_.read_checksum(r, g, p) == pay[p]
