"""CPU oracle of the reference data path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import
this package; the product (paper_2604_12171_b200) never does and has no CPU
fallback.  It wraps liboracle.so (oracle.c, a C restatement of
pipeshift/{events,kvstore,migrator}.py) behind the reference's Python API so
the same seeded op sequences (tests/opgen.py) can be replayed against the
reference (golden fixtures), the oracle, and the GPU store.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from math import ceil
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

OR_OK, OR_E_OVERFLOW, OR_E_BELOW_LIVE, OR_E_UNKNOWN_SLOT, OR_E_UNKNOWN_GROUP = 0, -1, -2, -3, -4
OR_E_INVALID = -6

_lib = None


def build() -> Path:
    src = [HERE / "oracle.c", HERE / "oracle.h", HERE / "llama_exact.c", HERE / "Makefile"]
    if not LIB.exists() or any(p.stat().st_mtime > LIB.stat().st_mtime for p in src):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        i32, i64, u64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
        sigs = {
            "or_crc32": (C.c_uint32, [vp, i64, C.c_uint32]),
            "or_stable_hash": (u64, [vp, i64]),
            "or_payload": (u64, [u64, i64]),
            "or_expand_word": (u64, [u64, C.c_uint32, C.c_uint32]),
            "or_expand_cell": (None, [u64, C.c_uint32, vp, i64]),
            "or_store_new": (vp, [C.c_int, C.c_int, C.c_int, i64, vp, C.c_int, C.c_int, i64]),
            "or_store_free": (None, [vp]),
            "or_last_error": (C.c_char_p, []),
            "or_capacity": (i64, [vp]), "or_used": (i64, [vp]), "or_occupied": (i64, [vp]),
            "or_resident": (C.c_int, [vp, vp, C.c_int]),
            "or_add_group": (C.c_int, [vp, C.c_int]),
            "or_append": (C.c_int, [vp, i32, C.c_int, i64, vp]),
            "or_write_slots": (C.c_int, [vp, i32, C.c_int, i64, vp, vp]),
            "or_read_checksum": (C.c_int, [vp, i32, C.c_int, i64, C.POINTER(u64)]),
            "or_read_cell": (C.c_int, [vp, i32, C.c_int, i64, C.c_int, vp]),
            "or_compact": (i64, [vp]),
            "or_resize": (C.c_int, [vp, i64]),
            "or_drop_groups": (C.c_int, [vp, vp, C.c_int, C.POINTER(i64)]),
            "or_free_request": (C.c_int, [vp, i32, vp, C.c_int]),
            "or_utilization": (C.c_double, [vp]),
            "or_blocks": (i64, [vp, vp, vp, i64]),
            "or_tables": (i64, [vp, vp, i64]),
            "or_chain": (i64, [vp, i32, vp, i64]),
            "or_written": (C.c_int, [vp, i32, vp, vp, C.c_int]),
            "or_block_occupied": (i64, [vp, i64]),
            "or_block_cells": (C.c_int, [vp, i64, C.c_int, vp, vp, C.c_int]),
            "or_dirty_new": (vp, []), "or_dirty_free": (None, [vp]),
            "or_dirty_mark": (None, [vp, i32, i32, i64, i64]),
            "or_dirty_count": (i64, [vp]),
            "or_dirty_discard": (i64, [vp, i32]),
            "or_dirty_drain": (i64, [vp, vp, i64, vp, vp, vp, i64]),
            "or_patch_round": (C.c_int, [vp, vp, vp, vp, i64, C.c_int, C.c_int,
                                         C.POINTER(i64), C.POINTER(i64)]),
            # llama_exact.c: the tiny Llama's exact-mode arithmetic
            "or_det_exp": (C.c_double, [C.c_double]),
            "or_bf16_round": (C.c_double, [C.c_double]),
            "or_ex_gemv": (None, [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int]),
            "or_ex_rmsnorm": (None, [vp, vp, vp, C.c_int, C.c_int, C.c_double]),
            "or_ex_rope": (None, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]),
            "or_ex_silu_mul": (None, [vp, vp, vp, i64]),
            "or_ex_attn": (None, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                  vp, vp]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data)


def stable_hash(*parts) -> int:
    data = "\x1f".join(str(p) for p in parts).encode()
    buf = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    return int(lib().or_stable_hash(_p(buf), len(data)))


def payload(seed: int, pos: int) -> int:
    return int(lib().or_payload(seed, pos))


def expand_cell(fp: int, layer: int, nbytes: int) -> bytes:
    out = np.zeros(nbytes, np.uint8)
    lib().or_expand_cell(fp, layer, _p(out), nbytes)
    return out.tobytes()


class KvError(Exception):
    pass


class KvOverflow(KvError):
    pass


class CapacityBelowLive(KvError):
    pass


class UnknownSlot(KvError):
    pass


class UnknownLayerGroup(KvError):
    pass


_EXC = {OR_E_OVERFLOW: KvOverflow, OR_E_BELOW_LIVE: CapacityBelowLive,
        OR_E_UNKNOWN_SLOT: UnknownSlot, OR_E_UNKNOWN_GROUP: UnknownLayerGroup,
        OR_E_INVALID: ValueError}


def _check(rc):
    if rc != OR_OK:
        raise _EXC.get(rc, RuntimeError)(lib().or_last_error().decode())


class Registry:
    def __init__(self):
        self.ids: dict = {}
        self.names: list = []

    def handle(self, rid) -> int:
        if rid not in self.ids:
            self.ids[rid] = len(self.names)
            self.names.append(rid)
        return self.ids[rid]

    def rank(self) -> np.ndarray:
        order = sorted(range(len(self.names)), key=lambda i: self.names[i])
        r = np.zeros(max(len(order), 1), np.int32)
        r[order] = np.arange(len(order), dtype=np.int32)
        return r


class _Block:
    def __init__(self, st, bid, owner):
        self._st, self.block_id, self._owner = st, bid, owner
        self.address = (st.gpu_id << 44) | (bid << 21)

    @property
    def state(self):
        return "live" if self._owner >= 0 else "free"

    def occupied_tokens(self):
        return int(lib().or_block_occupied(self._st._h, self.block_id))


class _Table:
    def __init__(self, st, h):
        self._st, self._h = st, h

    @property
    def written(self):
        return self._st._written(self._h)

    @property
    def chain(self):
        ids = np.zeros(4096, np.int64)
        n = lib().or_chain(self._st._h, self._h, _p(ids), len(ids))
        return [_Block(self._st, int(b), self._h) for b in ids[:n]]


class _Tables:
    def __init__(self, st):
        self._st = st

    def _handles(self):
        buf = np.zeros(4096, np.int32)
        n = lib().or_tables(self._st._h, _p(buf), len(buf))
        return [int(x) for x in buf[:n]]

    def __contains__(self, rid):
        h = self._st.reg.ids.get(rid)
        return h is not None and h in self._handles()

    def __getitem__(self, rid):
        if rid not in self:
            raise KeyError(rid)
        return _Table(self._st, self._st.reg.ids[rid])

    def __iter__(self):
        return iter([self._st.reg.names[h] for h in self._handles()])

    def __len__(self):
        return len(self._handles())


class OracleStore:
    """KvStore restated in C (kvstore.py:88-360); same Python surface."""

    def __init__(self, gpu_id, stacking_factor, tokens_per_block, capacity_blocks,
                 resident_groups=(), num_groups=64, cell_bytes=0, registry=None):
        g = np.asarray(sorted(set(resident_groups)) or [0], np.int32)
        n = len(set(resident_groups))
        h = lib().or_store_new(gpu_id, stacking_factor, tokens_per_block, capacity_blocks,
                               _p(g), n, num_groups, cell_bytes)
        if not h:
            raise ValueError(lib().or_last_error().decode())
        self._h = h
        self.gpu_id, self.stacking_factor, self.tokens_per_block = gpu_id, stacking_factor, tokens_per_block
        self.num_groups, self.cell_bytes = num_groups, cell_bytes
        self.reg = registry or Registry()
        self.tables = _Tables(self)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_store_free(self._h)
            self._h = None

    def _written(self, h):
        gs = np.zeros(self.num_groups, np.int32)
        cs = np.zeros(self.num_groups, np.int64)
        n = lib().or_written(self._h, h, _p(gs), _p(cs), self.num_groups)
        return {int(gs[i]): int(cs[i]) for i in range(n)}

    @property
    def resident_groups(self):
        buf = np.zeros(self.num_groups, np.int32)
        n = lib().or_resident(self._h, _p(buf), len(buf))
        return _ResidentProxy(self, {int(x) for x in buf[:n]})

    @resident_groups.setter
    def resident_groups(self, value):
        for g in set(value) - set(self.resident_groups):
            _check(lib().or_add_group(self._h, g))

    capacity_blocks = property(lambda self: int(lib().or_capacity(self._h)))
    used_blocks = property(lambda self: int(lib().or_used(self._h)))
    free_blocks = property(lambda self: self.capacity_blocks - self.used_blocks)
    occupied = property(lambda self: int(lib().or_occupied(self._h)))

    @property
    def blocks(self):
        n = self.capacity_blocks
        ids = np.zeros(max(n, 1), np.int64)
        own = np.zeros(max(n, 1), np.int32)
        lib().or_blocks(self._h, _p(ids), _p(own), n)
        return [_Block(self, int(ids[i]), int(own[i])) for i in range(n)]

    def append(self, rid, g, n, payloads):
        if n != len(payloads):
            raise ValueError("one checksum per token required")
        if n == 0:
            return []
        h = self.reg.handle(rid)
        pay = np.asarray([int(x) for x in payloads], np.uint64)
        _check(lib().or_append(self._h, h, g, n, _p(pay)))
        from types import SimpleNamespace
        end = self._written(h)[g]
        chain = _Table(self, h).chain
        s = self.tokens_per_block
        return [SimpleNamespace(block_id=chain[(end - n + i) // s].block_id, layer_group=g,
                                offset=(end - n + i) % s, checksum=int(payloads[i]))
                for i in range(n)]

    def write_slots(self, rid, g, items):
        if not items:
            return
        h = self.reg.handle(rid)
        pos = np.asarray([p for p, _ in items], np.int64)
        pay = np.asarray([int(c) for _, c in items], np.uint64)
        _check(lib().or_write_slots(self._h, h, g, len(items), _p(pos), _p(pay)))

    def read_checksum(self, rid, g, tok):
        h = self.reg.ids.get(rid)
        if h is None:
            raise UnknownSlot(rid)
        out = C.c_uint64()
        _check(lib().or_read_checksum(self._h, h, g, tok, C.byref(out)))
        return out.value

    def read_cell(self, rid, g, tok, layer):
        out = np.zeros(self.cell_bytes, np.uint8)
        _check(lib().or_read_cell(self._h, self.reg.ids[rid], g, tok, layer, _p(out)))
        return out.tobytes()

    def compact(self):
        return int(lib().or_compact(self._h))

    def resize(self, n):
        _check(lib().or_resize(self._h, n))

    def drop_layer_groups(self, groups):
        g = np.asarray(sorted(set(groups)) or [0], np.int32)
        out = C.c_int64()
        _check(lib().or_drop_groups(self._h, _p(g), len(set(groups)), C.byref(out)))
        return out.value

    def free_request(self, rid):
        h = self.reg.ids.get(rid)
        if h is None:
            return {}
        st = np.zeros(3 * 64, np.int64)
        n = lib().or_free_request(self._h, h, _p(st), 64)
        return {int(st[3 * i]): (int(st[3 * i + 1]), int(st[3 * i + 2])) for i in range(n)}

    def effective_utilization(self):
        return float(lib().or_utilization(self._h))

    def snapshot_group(self, g):
        out = {}
        for rid in sorted(self.tables):
            w = self.tables[rid].written.get(g, 0)
            if w:
                out[rid] = tuple(self.read_checksum(rid, g, p) for p in range(w))
        return out

    def state_digest(self):
        tables = []
        offs = np.zeros(4096, np.int64)
        fps = np.zeros(4096, np.uint64)
        for rid in sorted(self.tables):
            t = self.tables[rid]
            per_block = []
            for b in t.chain:
                cells = []
                for g in range(self.num_groups):
                    n = lib().or_block_cells(self._h, b.block_id, g, _p(offs), _p(fps), 4096)
                    if n > 0:
                        cells.append((g, tuple((int(offs[i]), int(fps[i])) for i in range(n))))
                per_block.append(tuple(cells))
            tables.append((rid, tuple(sorted(t.written.items())), tuple(per_block)))
        return (self.capacity_blocks, self.used_blocks, tuple(sorted(self.resident_groups)),
                tuple(tables))

    def blocks_needed(self, rid, extra):
        h = self.reg.ids.get(rid)
        w = self._written(h) if h is not None else {}
        have = len(_Table(self, h).chain) if h is not None and rid in self.tables else 0
        return max(0, ceil((max(w.values(), default=0) + extra) / self.tokens_per_block) - have)


class _ResidentProxy(set):
    def __init__(self, st, items):
        super().__init__(items)
        self._st = st

    def __ior__(self, other):
        for g in other:
            _check(lib().or_add_group(self._st._h, g))
        set.update(self, other)
        return self


class OracleDirty:
    """DirtyBitmap (migrator.py:24-48) over int handles."""

    def __init__(self):
        self._h = lib().or_dirty_new()

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_dirty_free(self._h)

    def mark(self, req, g, start, n):
        lib().or_dirty_mark(self._h, req, g, start, n)

    def __len__(self):
        return int(lib().or_dirty_count(self._h))

    def discard(self, req):
        return int(lib().or_dirty_discard(self._h, req))

    def drain(self, rank):
        n = len(self)
        r = np.zeros(max(n, 1), np.int32)
        g = np.zeros(max(n, 1), np.int32)
        p = np.zeros(max(n, 1), np.int64)
        m = lib().or_dirty_drain(self._h, _p(rank), len(rank), _p(r), _p(g), _p(p), max(n, 1))
        return [(int(r[i]), int(g[i]), int(p[i])) for i in range(m)]

    def patch_round(self, src, dst, rank, layers_per_group, threads=1):
        keys = C.c_int64()
        cells = C.c_int64()
        _check(lib().or_patch_round(self._h, src._h, dst._h, _p(rank), len(rank),
                                    layers_per_group, threads, C.byref(keys), C.byref(cells)))
        return keys.value, cells.value
