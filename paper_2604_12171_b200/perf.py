"""Perf-mode drivers of the live-reconfiguration data path (no simulated clock).

Used by bench.py and the GPU tests.  Everything here calls the C-ABI directly
with device-resident buffers; the parity-mode classes (kvstore/migrator) are
the same native objects driven by the reference's event clock instead.

Workload (BASELINE configs[1]): Llama-3-8B shape -- 32 layers, 32 q heads,
8 KV heads x 128, bf16 -> 4096 B of KV per token per layer; stacking k = 4,
16-token blocks; one PP2 stage holds layers 1-16 (groups 0-3); the PP2->4
split moves layers 9-16 (groups 2-3) to a new stage; B = 256 live requests at
2048 tokens of context.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from math import ceil

import numpy as np

from . import _native as N
from .events import stable_hash
from .kvstore import KvStore, RequestRegistry


@dataclass
class Workload:
    name: str = "llama3-8b PP2->4: one migrating pair (layers 9-16), B=256, ctx=2048"
    n_layers: int = 32
    n_q: int = 32
    n_kv: int = 8
    head_dim: int = 128
    k: int = 4
    s: int = 16
    batch: int = 256
    ctx: int = 2048
    src_groups: tuple = (0, 1, 2, 3)
    mig_groups: tuple = (2, 3)

    @property
    def cell_bytes(self) -> int:
        return 2 * self.n_kv * self.head_dim * 2

    @property
    def blocks_per_req(self) -> int:
        return ceil(self.ctx / self.s)

    @property
    def payload_bytes(self) -> int:
        """KvPatch.payload_bytes of the bulk round: cells x token_kv_bytes (migrator.py:70-71)."""
        return self.batch * self.ctx * len(self.mig_groups) * self.k * self.cell_bytes

    @property
    def model_groups(self) -> int:
        return self.n_layers // self.k


def rid(i: int) -> str:
    return f"r{i:04d}"


def append_batch(store: KvStore, reqs: list[int], groups: list[int], counts: list[int],
                 seeds: list[int], kv_dev: int | None = None, mark: bool = False) -> int:
    r = N.as_i32(reqs)
    g = N.as_i32(groups)
    c = N.as_i64(counts)
    sd = N.as_u64(seeds)
    done = C.c_int()
    if kv_dev is not None:
        store.wait_for_caller_stream()
    rc = N.lib().pl_store_append_batch(store._h, len(reqs), N.ptr(r), N.ptr(g), N.ptr(c),
                                       N.ptr(sd), None, kv_dev, 1 if mark else 0, C.byref(done),
                                       None, 0)
    N.check(rc)
    return done.value


def append_batch_payloads(store: KvStore, reqs: list[int], groups: list[int], counts: list[int],
                          payloads: np.ndarray, mark: bool = False) -> int:
    """KvStore.append(rid, group, n, payloads) for many items in one call: host payloads
    (uint64, items concatenated) -> one H2D + one K1 launch."""
    r, g, c = N.as_i32(reqs), N.as_i32(groups), N.as_i64(counts)
    pl = np.ascontiguousarray(payloads, dtype=np.uint64)
    done = C.c_int()
    N.check(N.lib().pl_store_append_batch_payloads(store._h, len(r), N.ptr(r), N.ptr(g), N.ptr(c),
                                                   N.ptr(pl), 1 if mark else 0, C.byref(done)))
    return done.value


def engine_payloads(seed: int, n: int) -> np.ndarray:
    """PipelineEngine._payloads (engine.py:252-261) for positions 0..n-1, vectorised:
    (seed * 0x9E3779B97F4A7C15 + pos * 0xBF58476D1CE4E5B9) mod 2^64, top bit cleared."""
    pos = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        v = np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15) + pos * np.uint64(0xBF58476D1CE4E5B9)
    return v & np.uint64((1 << 63) - 1)


class NativePatch:
    """A pl_patch handle for perf runs (the parity-mode owner is MigrationStream)."""

    def __init__(self, src: KvStore, groups, layers_per_group: int) -> None:
        g = N.as_i32(list(groups))
        lpg = N.as_i32([layers_per_group] * len(groups))
        h = C.c_void_p()
        N.check(N.lib().pl_patch_create(src._h, N.ptr(g), N.ptr(lpg), len(groups), C.byref(h)))
        self.h = h
        self.src = src
        self._rank, self._rank_args = None, (None, 0)
        self._keys, self._cells = C.c_int64(), C.c_int64()
        self._keys_ref, self._cells_ref = C.byref(self._keys), C.byref(self._cells)
        self._push_fn, self._push_args = N.lib().pl_patch_push, (None, None)
        N.check(N.lib().pl_patch_set_active(h, 1))

    def seed(self) -> int:
        out = C.c_int64()
        N.check(N.lib().pl_patch_seed(self.h, C.byref(out)))
        return out.value

    def push(self, dst: KvStore, rank: np.ndarray) -> tuple[int, int]:
        # ctypes argument objects are built once per rank array: numpy's .ctypes costs ~2 us,
        # as much as a steady round's whole host enqueue
        # (and the whole argument tuple once per (destination, rank): a steady round's
        # Python side is then one foreign call)
        if self._rank is not rank or self._push_args[0] is not dst:
            self._rank, self._rank_args = rank, (N.ptr(rank), len(rank))
            self._push_args = (dst, (self.h, dst._h, *self._rank_args, self._keys_ref,
                                     self._cells_ref))
        rc = self._push_fn(*self._push_args[1])
        if rc:
            N.check(rc)
        return self._keys.value, self._cells.value

    def stream_ptr(self) -> int:
        """The stream this pair's K3/K4/K5 are enqueued on."""
        out = C.c_void_p()
        N.check(N.lib().pl_patch_stream(self.h, C.byref(out)))
        return out.value or 0

    def last_push_stats(self) -> dict:
        """Host phases of the last push (ms), pl_patch_last_push_stats."""
        out = np.zeros(8, dtype=np.float64)
        N.check(N.lib().pl_patch_last_push_stats(self.h, N.ptr(out)))
        keys = ("adopt_wait", "snapshot", "reserve", "dst_flush", "k3_enqueue", "copy_enqueue",
                "total")
        d = {k: round(float(v), 4) for k, v in zip(keys, out)}
        d["chunked"] = bool(out[7] == 1)
        # launch-first steady round: the destination's host bookkeeping ran on the worker
        # thread ("reserve" is then the worker's time, off the caller's path)
        d["async_bookkeeping"] = bool(out[7] == 2)
        return d

    def mark_batch(self, reqs, groups, starts, counts) -> None:
        r, g = N.as_i32(reqs), N.as_i32(groups)
        st, c = N.as_i64(starts), N.as_i64(counts)
        N.check(N.lib().pl_patch_mark_batch(self.h, len(r), N.ptr(r), N.ptr(g), N.ptr(st),
                                            N.ptr(c)))

    def discard_request(self, rid, registry) -> int:
        """DirtyBitmap.discard_request (migrator.py:43-48) for a finished request."""
        h = registry.find(rid)
        if h is None:
            return 0
        out = C.c_int64()
        N.check(N.lib().pl_patch_discard_request(self.h, h, C.byref(out)))
        return out.value

    def set_stream(self, stream_ptr: int | None) -> None:
        """K3/K4/K5 of this pair on a side stream (overlapped with decode)."""
        N.check(N.lib().pl_patch_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def dirty_keys(self) -> int:
        out = C.c_int64()
        N.check(N.lib().pl_patch_dirty_keys(self.h, C.byref(out)))
        return out.value

    def device_drained(self) -> int:
        out = C.c_int64()
        N.check(N.lib().pl_patch_device_drained(self.h, C.byref(out)))
        return out.value

    def close(self) -> None:
        if self.h is not None:
            N.lib().pl_patch_destroy(self.h)
            self.h = None


@dataclass
class PatchRig:
    """Source stage store filled with B x ctx tokens in every group, destination store
    holding the migrating groups, and the pair's native patch engine."""

    wl: Workload
    device: int = 0
    registry: RequestRegistry = field(default_factory=RequestRegistry)

    def __post_init__(self) -> None:
        wl = self.wl
        cap = wl.batch * (wl.blocks_per_req + 2) + 64
        self.src = KvStore(1, wl.k, wl.s, cap, wl.src_groups, num_groups=wl.model_groups,
                           cell_bytes=wl.cell_bytes, device=self.device, registry=self.registry)
        self.dst = KvStore(2, wl.k, wl.s, cap, (), num_groups=wl.model_groups,
                           cell_bytes=wl.cell_bytes, device=self.device, registry=self.registry)
        self.dst.resident_groups |= set(wl.mig_groups)
        self.handles = [self.registry.handle(rid(i)) for i in range(wl.batch)]
        self.patch = NativePatch(self.src, wl.mig_groups, wl.k)

    def use_stream(self, stream_ptr: int) -> None:
        for st in (self.src, self.dst):
            N.check(N.lib().pl_store_set_stream(st._h, C.c_void_p(stream_ptr)))

    def fill(self) -> None:
        wl = self.wl
        reqs, groups, counts, seeds = [], [], [], []
        for i in range(wl.batch):
            for g in wl.src_groups:
                reqs.append(self.handles[i])
                groups.append(g)
                counts.append(wl.ctx)
                seeds.append(stable_hash(rid(i), g))
        append_batch(self.src, reqs, groups, counts, seeds)
        self.src.sync()

    def bulk_round(self) -> tuple[int, int]:
        """one step: seed every live cell of the migrating groups, drain + push it"""
        self.patch.seed()
        return self.patch.push(self.dst, self.registry.rank())

    def close(self) -> None:
        self.patch.close()

    def destroy(self) -> None:
        self.close()
        self.src.close()
        self.dst.close()


def c2_live(rig: "PatchRig", stream, steps: int = 6) -> dict:
    """BASELINE configs[1] as a timeline: the PP2 stage keeps decoding (every step: K1
    appends one token per request to each of its 4 groups with the fused dirty mark, then
    K2 over its 16 layers) while the pair's patch engine runs on a low-priority side
    stream: the bulk copy of the two migrating groups, then one patch round per step.
    Reports decode ms/step before / during the bulk copy / during steady patching, the
    bulk copy's duration, and the switch pause (drain the decode stream, residual round,
    barrier).  Decode and patching share HBM, so the interference is the measured cost of
    live migration."""
    import torch

    wl = rig.wl
    lib = N.lib()
    dev = torch.device("cuda", rig.device)
    lo, _ = torch.cuda.Stream.priority_range()
    side = torch.cuda.Stream(device=rig.device, priority=lo)
    rig.patch.set_stream(side.cuda_stream)
    # the destination stage has its own stream (it is another GPU on hardware): its wait
    # for the applied patch must not block this stage's decode stream
    dst_stream = torch.cuda.Stream(device=rig.device)
    N.check(N.lib().pl_store_set_stream(rig.dst._h, C.c_void_p(dst_stream.cuda_stream)))
    B = wl.batch
    rows = torch.tensor(rig.handles, dtype=torch.int32, device=dev)
    ctx_now = [rig.src.tables[rid(i)].written.get(wl.src_groups[0], 0) for i in range(B)]
    q = torch.randn(B, wl.n_q, wl.head_dim, dtype=torch.bfloat16, device=dev)
    out = torch.empty_like(q)
    torch.cuda.synchronize(dev)   # produced on torch's stream, read on the stage's stream
    reqs = [h for h in rig.handles for _ in wl.src_groups]
    groups = [g for _ in rig.handles for g in wl.src_groups]
    seeds = [stable_hash(rid(i), g) for i in range(B) for g in wl.src_groups]

    def decode_step(mark: bool) -> float:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        append_batch(rig.src, reqs, groups, [1] * len(reqs), seeds, mark=mark)
        for i in range(B):
            ctx_now[i] += 1
        ctx = torch.tensor(ctx_now, dtype=torch.int32, device=dev)
        for g in wl.src_groups:
            for j in range(wl.k):
                N.check(lib.pl_paged_attn_decode(rig.src._h, g, j, C.c_void_p(q.data_ptr()),
                                                 C.c_void_p(out.data_ptr()),
                                                 C.c_void_p(rows.data_ptr()),
                                                 C.c_void_p(ctx.data_ptr()), B, wl.n_q, wl.n_kv,
                                                 wl.head_dim, wl.head_dim ** -0.5, max(ctx_now),
                                                 C.c_void_p(stream.cuda_stream)))
        e1.record(stream)
        return (e0, e1)

    torch.cuda.synchronize()
    base = [decode_step(False) for _ in range(steps)]
    torch.cuda.synchronize()
    base_ms = [a.elapsed_time(b) for a, b in base]
    # start: seed every live cell of the migrating groups, first round = bulk copy; decode
    # keeps stepping; the steps overlapping the bulk are found from the event timestamps
    rig.patch.seed()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    anchor = torch.cuda.Event(enable_timing=True)
    anchor.record(stream)
    side.wait_event(anchor)
    b0.record(side)
    th0 = time.perf_counter()
    keys, cells = rig.patch.push(rig.dst, rig.registry.rank())
    host_ms = (time.perf_counter() - th0) * 1e3
    push_phases = rig.patch.last_push_stats()
    b1.record(side)
    bulk_payload = cells * wl.cell_bytes
    during = [decode_step(True) for _ in range(steps)]
    torch.cuda.synchronize()
    assert rig.patch.device_drained() == keys, (rig.patch.device_drained(), keys)
    bulk_end = anchor.elapsed_time(b1)
    bulk_ms = b0.elapsed_time(b1)
    overlap = [(a, b) for a, b in during if anchor.elapsed_time(a) < bulk_end]
    during_ms = [a.elapsed_time(b) for a, b in overlap]
    steady, round_keys = [], []
    for _ in range(steps):
        k2, _ = rig.patch.push(rig.dst, rig.registry.rank())   # previous step's writes
        round_keys.append(k2)
        steady.append(decode_step(True))
    torch.cuda.synchronize()
    steady_ms = [a.elapsed_time(b) for a, b in steady]
    # switch: pause admission -> drain the in-flight step -> residual round -> barrier
    decode_step(True)
    t0 = time.perf_counter()
    stream.synchronize()                  # the in-flight decode step drains
    t1 = time.perf_counter()
    keys_res, cells_res = rig.patch.push(rig.dst, rig.registry.rank())
    side.synchronize()
    rig.dst.sync()                        # barrier: residual applied on the destination
    pause_ms = (time.perf_counter() - t0) * 1e3
    drain_ms = (t1 - t0) * 1e3
    rig.patch.set_stream(None)
    N.check(N.lib().pl_store_set_stream(rig.dst._h, C.c_void_p(stream.cuda_stream)))
    med = lambda xs: round(float(np.median(xs)), 4) if xs else None  # noqa: E731
    return {"decode_ms_per_step_alone": med(base_ms),
            "decode_ms_per_step_during_bulk": med(during_ms),
            "decode_steps_overlapping_bulk": len(during_ms),
            "decode_ms_per_step_steady_patching": med(steady_ms),
            "bulk": {"payload_bytes": bulk_payload, "ms": round(bulk_ms, 3),
                     "gbs": round(bulk_payload / bulk_ms / 1e6, 1),
                     "host_enqueue_ms": round(host_ms, 3), "host_phases_ms": push_phases},
            "steady_round_keys": round_keys[-1] if round_keys else 0,
            "switch_pause_ms": round(pause_ms, 4),
            "switch_pause_breakdown_ms": {"drain_in_flight_step": round(drain_ms, 4),
                                          "residual_patch_and_barrier": round(pause_ms - drain_ms, 4)},
            "residual_keys": keys_res,
            "residual_bytes": cells_res * wl.cell_bytes,
            "note": "decode (K1+K2, store stream) and patching (K3+K4+K5, low-priority side "
                    "stream) overlap on one GPU and share its HBM"}


def c3_live_resize(device: int = 0, fill_reqs: int = 703, ctx: int = 2040,
                   check: bool = False) -> dict:
    """BASELINE configs[2] at one GPU: the source stage of a Llama-3-70B PP 4 -> 8 boundary
    shift with HBM pre-filled by KV cache.

    Geometry from the reference's own max_blocks (cluster.py:180-201) with M = 180 GB,
    u = 0.9, 16-token blocks, k = 4 (unit 256 KiB + header): the stage holds layers 1-20
    (5 groups) at B = max_blocks(20) = 97,488 blocks.  In the target it keeps layers 1-12,
    sends 13-20 (groups 3, 4) to a new GPU and receives layers 21-24 (group 5) from its
    neighbour, so |C_cur u C_tgt| = 24 layers and Phase 2 must shrink to
    b_shrink = max_blocks(24) = 76,888 (coordinator.py:103-110, 189-201) while ~17 GB
    of live KV sits above that line; after the commit it drops groups 3, 4 and grows to
    b_new = max_blocks(16) = 128,387 (coordinator.py:340-354).  The migrating groups are
    pushed to a destination store on the same GPU (HBM-bound here, NVLink across GPUs).

    ``check`` (tests only; off in the bench): sampled fingerprints and cell bytes are read
    before the shrink and must survive the K6 relocation, the drop and the grow; the
    destination's migrating groups must equal the source's after the patch rounds."""
    import random

    import torch

    from .cluster import GpuSpec, ModelSpec, max_blocks

    gran = 16 * 4096 * 4
    gpu = GpuSpec(1, 180 * 10 ** 9 // gran * gran, 8e12, 1e-6, 1e-6, gran)
    model = ModelSpec(80, 1_711_000_000, 4096, 4)
    b_cur, b_shrink, b_new = (max_blocks(gpu, n, model, 0.9) for n in (20, 24, 16))
    reg = RequestRegistry()
    out: dict = {"b_cur": b_cur, "b_shrink": b_shrink, "b_new": b_new}
    src = KvStore(1, 4, 16, b_cur, (0, 1, 2, 3, 4), num_groups=20, cell_bytes=4096,
                  device=device, registry=reg)
    per_req = ceil(ctx / 16)
    hs = [reg.handle(rid(i)) for i in range(fill_reqs)]
    for c0 in range(0, fill_reqs, 64):
        chunk = hs[c0:c0 + 64]
        append_batch(src, [h for h in chunk for _ in range(5)], [g for _ in chunk for g in range(5)],
                     [ctx] * (5 * len(chunk)),
                     [stable_hash(rid(c0 + i), g) for i in range(len(chunk)) for g in range(5)])
    src.sync()
    # holes in the low slots: the shrink must relocate the live blocks above b_shrink
    freed = 0
    i = 0
    while src.used_blocks > b_shrink - 256:
        src.free_request(rid(i))
        freed += 1
        i += 2
    src.sync()
    torch.cuda.synchronize(device)
    out["filled_blocks"] = fill_reqs * per_req
    out["live_blocks"] = src.used_blocks
    out["kv_bytes_live"] = src.used_blocks * 5 * src.info()["unit_bytes"]
    samples = {}
    if check:
        rng = random.Random(2)
        live_ids = [i for i in range(fill_reqs) if src._has_table(hs[i])]
        for _ in range(96):
            i, g, p, j = rng.choice(live_ids), rng.randrange(5), rng.randrange(ctx), rng.randrange(4)
            samples[(rid(i), g, p, j)] = (src.read_checksum(rid(i), g, p), src.read_cell(rid(i), g, p, j))

    seeds = {(rid(i), g): stable_hash(rid(i), g) for i in range(fill_reqs) for g in range(5)}

    def verify(store, groups, what):
        for (r, g, p, j), (fp, cell) in samples.items():
            if g in groups:
                assert store.read_checksum(r, g, p) == fp, (what, r, g, p)
                assert store.read_cell(r, g, p, j) == cell, (what, r, g, p, j)
        out.setdefault("checks", []).append(what)
        # every live cell on the device (csrc/verify.cu), not just the samples
        v = store.verify_cells(seeds)
        out.setdefault("full_checks", []).append(
            {"what": what, "cells": v["cells"], "bad": v["bad_bytes"] + v["bad_fingerprints"]})

    # Phase 2: compact + shrink with relocation, then map the incoming group 5
    t0 = time.perf_counter()
    src.compact()
    src.resize(b_shrink)
    src.sync()
    out["phase2_shrink_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    out["phase2_shrink_stats"] = src.last_resize_stats()
    # full latency: until the retired tail is unmapped and back with the driver
    src.reclaim()
    out["phase2_shrink_full_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    if check:
        assert src.capacity_blocks == b_shrink and src.used_blocks == out["live_blocks"]
        verify(src, range(5), "relocation")
    free_gb = lambda: round(torch.cuda.mem_get_info(device)[0] / 1e9, 1)  # noqa: E731
    out["free_gb_after_shrink"] = free_gb()
    t0 = time.perf_counter()
    src.resident_groups.add(5)
    src.sync()
    out["map_incoming_group_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    # the pool itself is mapped on the reclaimer thread (lazy materialisation); Phase 3
    # starts after weight loading, by when it is done -- time it, outside the patch rounds
    out["map_incoming_group_background_ms"] = round(
        (time.perf_counter() - t0) * 1e3 + src.prepare_wait(), 3)
    out["map_incoming_group_full_ms"] = out["map_incoming_group_background_ms"]
    # Phase 3: bulk + one decode round of the two leaving groups
    dst = KvStore(2, 4, 16, src.used_blocks + 256, (), num_groups=20, cell_bytes=4096,
                  device=device, registry=reg)
    dst.resident_groups |= {3, 4}
    dst.prepare_wait()   # the destination's pools are mapped before its Phase 3, as above
    patch = NativePatch(src, (3, 4), 4)
    patch.seed()
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    keys, cells = patch.push(dst, reg.rank())
    src.sync()
    dst.sync()
    t = time.perf_counter() - t0
    out["bulk_patch"] = {"keys": keys, "payload_bytes": cells * 4096, "ms": round(t * 1e3, 3),
                         "gbs": round(cells * 4096 / t / 1e9, 1)}
    live = [h for h in hs if src._has_table(h)]
    names = [reg.name(h) for h in live]
    append_batch(src, [h for h in live for _ in range(5)], [g for _ in live for g in (0, 1, 2, 3, 4)],
                 [1] * (5 * len(live)), [stable_hash(n, g) for n in names for g in range(5)],
                 mark=True)
    src.sync()
    t0 = time.perf_counter()
    keys, cells = patch.push(dst, reg.rank())
    src.sync()
    dst.sync()
    out["residual_patch"] = {"keys": keys, "ms": round((time.perf_counter() - t0) * 1e3, 3)}
    if check:
        for g in (3, 4):
            assert dst.snapshot_group(g) == src.snapshot_group(g), g
        c = src.compare_cells(dst, (3, 4), [reg.name(h) for h in live])
        assert c["missing"] == 0
        out.setdefault("full_checks", []).append(
            {"what": "patched", "cells": c["cells"], "bad": c["bad_positions"]})
        verify(dst, (3, 4), "patched(dst)")
    patch.close()
    out["free_gb_during_patch"] = free_gb()
    dst.close()   # the destination is another GPU on hardware; free its HBM here
    # post-commit: drop the leaving groups, grow to b_new (re-maps their chunks)
    v0 = src.vmm_stats()
    t0 = time.perf_counter()
    src.drop_layer_groups([3, 4])
    out["drop_groups_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    # the drop's full latency (unmap of the groups' pools) is not forced here: post-commit
    # cleanup grows right after, re-mapping those chunks (vmm.cu); the grow's full latency
    # below includes that work
    t0 = time.perf_counter()
    src.resize(b_new)
    src.sync()
    out["grow_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    # lazy grow: the tail is mapped on the reclaimer thread; time until that is done
    out["grow_background_ms"] = round((time.perf_counter() - t0) * 1e3 + src.prepare_wait(), 3)
    out["grow_full_ms"] = out["grow_background_ms"]
    if check:
        assert src.capacity_blocks == b_new
        verify(src, (0, 1, 2), "drop+grow")
    v1 = src.vmm_stats()
    out["grow_stats"] = {**src.last_resize_stats(),
                         **{k: v1[k] - v0[k] for k in ("tail_reused_chunks", "cache_reused_chunks",
                                                      "created_chunks")}}
    out["mapped_bytes_end"] = src.info()["mapped_bytes"]
    src.reclaim()
    src.close()
    return out


def c5_sweep(device: int = 0, rates=(0.01, 0.05, 0.25, 1.0), block_sizes=(8, 16, 32, 64, 128),
             batch: int = 64, ctx: int = 2048, rounds: int = 8, seed: int = 0) -> list[dict]:
    """BASELINE configs[4] at one GPU: dirty-rate x block-size sweep of the patch round.

    Per block size: a source stage with ``batch`` requests x ``ctx`` tokens in two
    migrating k=4 groups (Llama-3 cells, 4096 B), a destination holding those groups, and
    one patch engine.  Per dirty rate: uniform-random (request, group, position) keys,
    seeded, are marked (outside the timed region), then one round = drain (K3) + fused
    gather/scatter push (K4+K5) is timed wall-clock with the device synchronised on
    both sides.  Plus the structured decode pattern: one key per live request and group
    (the newest token).  Source and destination share the GPU, so the bound is HBM
    (payload read + write), not NVLink.  ``ms`` is the round's wall time (host block
    manager + launches + device), ``kernel_ms`` the K3 + fused-push kernels alone."""
    import torch

    rng = np.random.default_rng(seed)
    out = []
    k, cell = 4, 4096
    for s in block_sizes:
        reg = RequestRegistry()
        blocks = batch * (ceil(ctx / s) + 1) + 16
        src = KvStore(1, k, s, blocks, (0, 1), num_groups=2, cell_bytes=cell, device=device,
                      registry=reg)
        dst = KvStore(2, k, s, blocks, (0, 1), num_groups=2, cell_bytes=cell, device=device,
                      registry=reg)
        hs = [reg.handle(rid(i)) for i in range(batch)]
        reqs = [h for h in hs for _ in (0, 1)]
        groups = [g for _ in hs for g in (0, 1)]
        append_batch(src, reqs, groups, [ctx] * len(reqs),
                     [stable_hash(rid(i), g) for i in range(batch) for g in (0, 1)])
        patch = NativePatch(src, (0, 1), k)
        patch.seed()
        patch.push(dst, reg.rank())   # bulk copy: destination chains exist from here on
        src.sync()
        dst.sync()
        rank = reg.rank()
        cases = [("decode", None)] + [(f"{r:g}", r) for r in rates]
        for name, r in cases:
            times, dev, book, keys_n = [], [], [], 0
            # wall rounds first (kernel timing off: its event pairs would sit on the host
            # path), then the same number of rounds with the kernels timed
            for it in range(2 * (rounds + 1)):
                timed = it > rounds
                if r is None:
                    rq, gq, st = reqs, groups, [ctx - 1] * len(reqs)
                else:
                    n_keys = max(1, int(round(r * batch * 2 * ctx)))
                    flat = rng.choice(batch * 2 * ctx, size=n_keys, replace=False)
                    rq = [hs[x // (2 * ctx)] for x in flat]
                    gq = [int((x // ctx) % 2) for x in flat]
                    st = [int(x % ctx) for x in flat]
                patch.mark_batch(rq, gq, st, [1] * len(rq))
                src.sync()
                torch.cuda.synchronize(device)
                if timed:
                    N.check(N.lib().pl_timing_reset())
                    N.check(N.lib().pl_timing_enable(1))
                t0 = time.perf_counter()
                keys, cells = patch.push(dst, rank)
                # the destination's stream waits on the round's copy (ev_applied): its sync
                # is the round's end on the device
                dst.sync()
                t1 = time.perf_counter()
                src.sync()
                if timed:
                    N.check(N.lib().pl_timing_enable(0))
                    dev.append(N.timing("drain")[0] + N.timing("patch_push")[0]
                               + N.timing("drain_push")[0])
                elif it > 0:
                    times.append(t1 - t0)
                    book.append(patch.last_push_stats()["reserve"])
                keys_n = keys
            times = [0.0] + times   # (the first wall round is warm-up)
            t = float(np.median(times[1:]))
            td = float(np.median(dev)) / 1e3
            payload = keys_n * k * cell
            out.append({"tokens_per_block": s, "dirty": name, "keys": keys_n,
                        "payload_bytes": payload, "ms": round(t * 1e3, 4),
                        "gbs": round(payload / t / 1e9, 2),
                        "hbm_gbs": round(2 * (payload + 8 * keys_n) / t / 1e9, 2),
                        "kernel_ms": round(td * 1e3, 4),
                        # destination write_slots bookkeeping, on the host worker thread for
                        # launch-first rounds (off the round's wall time)
                        "host_bookkeeping_ms": round(float(np.median(book)), 4),
                        "kernel_hbm_gbs": round(2 * (payload + 8 * keys_n) / td / 1e9, 2) if td else None})
        patch.close()
        del src, dst
    return out


def c5_pairs(device: int = 0, pairs=(1, 2, 4, 7), batch: int = 32, ctx: int = 2048,
             rounds: int = 3) -> list[dict]:
    """BASELINE configs[4]'s concurrent-pairs axis at one GPU: P distinct (src, dst) pairs,
    each with its own stores and its own low-priority patch stream, push their bulk round
    at the same time (one host thread enqueues all P, then the device runs them
    concurrently).  All pairs share one GPU's HBM here, so the aggregate should hold at
    the single-pair HBM rate whatever P is -- i.e. the engine adds no serialisation;
    across GPUs each distinct-source pair would get its own NVLink."""
    import torch

    wl = Workload(batch=batch, ctx=ctx)
    lo, _ = torch.cuda.Stream.priority_range()
    out = []
    for P in pairs:
        rigs, streams = [], []
        for _ in range(P):
            rig = PatchRig(wl, device=device)
            rig.fill()
            st = torch.cuda.Stream(device=device, priority=lo)
            rig.patch.set_stream(st.cuda_stream)
            rigs.append(rig)
            streams.append(st)
        for rig in rigs:                       # cold round: destination chains exist after it
            rig.bulk_round()
        torch.cuda.synchronize(device)
        times = []
        for _ in range(rounds):
            for rig in rigs:
                rig.patch.seed()
            torch.cuda.synchronize(device)
            t0 = time.perf_counter()
            for rig in rigs:
                rig.patch.push(rig.dst, rig.registry.rank())
            torch.cuda.synchronize(device)
            times.append(time.perf_counter() - t0)
        t = float(np.median(times))
        payload = P * wl.payload_bytes
        out.append({"pairs": P, "payload_bytes": payload, "ms": round(t * 1e3, 3),
                    "aggregate_gbs": round(payload / t / 1e9, 1),
                    "per_pair_gbs": round(payload / P / t / 1e9, 1)})
        for rig in rigs:
            rig.destroy()
        del rigs, streams
        torch.cuda.synchronize(device)
    return out


def read_peaks(path) -> dict:
    import json
    try:
        return json.loads(open(path).read())
    except Exception:
        return {}


def now() -> float:
    return time.perf_counter()
