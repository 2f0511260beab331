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
    rc = N.lib().pl_store_append_batch(store._h, len(reqs), N.ptr(r), N.ptr(g), N.ptr(c),
                                       N.ptr(sd), None, kv_dev, 1 if mark else 0, C.byref(done),
                                       None, 0)
    N.check(rc)
    return done.value


class NativePatch:
    """A pl_patch handle for perf runs (the parity-mode owner is MigrationStream)."""

    def __init__(self, src: KvStore, groups, layers_per_group: int) -> None:
        g = N.as_i32(list(groups))
        lpg = N.as_i32([layers_per_group] * len(groups))
        h = C.c_void_p()
        N.check(N.lib().pl_patch_create(src._h, N.ptr(g), N.ptr(lpg), len(groups), C.byref(h)))
        self.h = h
        self.src = src
        N.check(N.lib().pl_patch_set_active(h, 1))

    def seed(self) -> int:
        out = C.c_int64()
        N.check(N.lib().pl_patch_seed(self.h, C.byref(out)))
        return out.value

    def push(self, dst: KvStore, rank: np.ndarray) -> tuple[int, int]:
        keys, cells = C.c_int64(), C.c_int64()
        N.check(N.lib().pl_patch_push(self.h, dst._h, N.ptr(rank), len(rank), C.byref(keys),
                                      C.byref(cells)))
        return keys.value, cells.value

    def mark_batch(self, reqs, groups, starts, counts) -> None:
        r, g = N.as_i32(reqs), N.as_i32(groups)
        st, c = N.as_i64(starts), N.as_i64(counts)
        N.check(N.lib().pl_patch_mark_batch(self.h, len(r), N.ptr(r), N.ptr(g), N.ptr(st),
                                            N.ptr(c)))

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


def c5_sweep(device: int = 0, rates=(0.01, 0.05, 0.25, 1.0), block_sizes=(8, 16, 32, 64, 128),
             batch: int = 64, ctx: int = 2048, rounds: int = 3, seed: int = 0) -> list[dict]:
    """BASELINE configs[4] at one GPU: dirty-rate x block-size sweep of the patch round.

    Per block size: a source stage with ``batch`` requests x ``ctx`` tokens in two
    migrating k=4 groups (Llama-3 cells, 4096 B), a destination holding those groups, and
    one patch engine.  Per dirty rate: uniform-random (request, group, position) keys,
    seeded, are marked (outside the timed region), then one round = drain (K3) + fused
    gather/scatter push (K4+K5) is timed wall-clock with the device synchronised on
    both sides.  Plus the structured decode pattern: one key per live request and group
    (the newest token).  Source and destination share the GPU, so the bound is HBM
    (payload read + write), not NVLink."""
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
            times, keys_n = [], 0
            for _ in range(rounds + 1):
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
                t0 = time.perf_counter()
                keys, cells = patch.push(dst, rank)
                dst.sync()
                src.sync()
                times.append(time.perf_counter() - t0)
                keys_n = keys
            t = float(np.median(times[1:]))
            payload = keys_n * k * cell
            out.append({"tokens_per_block": s, "dirty": name, "keys": keys_n,
                        "payload_bytes": payload, "ms": round(t * 1e3, 4),
                        "gbs": round(payload / t / 1e9, 2),
                        "hbm_gbs": round(2 * (payload + 8 * keys_n) / t / 1e9, 2)})
        patch.close()
        del src, dst
    return out


def read_peaks(path) -> dict:
    import json
    try:
        return json.loads(open(path).read())
    except Exception:
        return {}


def now() -> float:
    return time.perf_counter()
