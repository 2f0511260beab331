"""GPU-backed KV block manager: the drop-in for pipeshift.kvstore.

Same public surface as /root/reference/pkg/src/pipeshift/kvstore.py
(KvStore, kv_init, StackedSlot, the exception classes), implemented over the
C-ABI of libpipelive.so: block ids, chains and occupancy follow the
reference's exact policy in the native host runtime, while every KV cell,
fingerprint header and block table lives in HBM and is written by the sm_100a
kernels.  There is no CPU fallback: constructing a store without the native
library or a CUDA device raises NativeUnavailable.

Layout: one VMM-backed pool per layer group; a (block, group)
unit is [fingerprint header: s x u64][layer 0: s cells]...[layer k-1: s cells];
a cell is ``cell_bytes`` of one token of one layer.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from math import ceil
from typing import Iterable, Iterator, Sequence

import numpy as np

from . import _native as N
from .cluster import GpuSpec, ModelSpec


class KvError(Exception):
    pass


class KvOverflow(KvError):
    """No free block available for the requested append (kvstore.py:27-28)."""


class CapacityBelowLive(KvError):
    """Shrink target below the number of live blocks (kvstore.py:31-32)."""


class UnknownSlot(KvError):
    pass


class UnknownLayerGroup(KvError):
    pass


class InsufficientMemory(KvError):
    pass


_ERRORS = {
    N.PL_E_KV_OVERFLOW: KvOverflow,
    N.PL_E_CAPACITY_BELOW_LIVE: CapacityBelowLive,
    N.PL_E_UNKNOWN_SLOT: UnknownSlot,
    N.PL_E_UNKNOWN_LAYER_GROUP: UnknownLayerGroup,
    N.PL_E_INSUFFICIENT_MEMORY: InsufficientMemory,
    N.PL_E_INVALID: ValueError,
}


def _check(rc: int) -> None:
    if rc != N.PL_OK:
        msg = N.lib().pl_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, N.NativeError)(msg) if rc in _ERRORS else N.NativeError(rc, msg)


#: bytes stored per (token, layer) cell when the caller does not say: parity
#: runs keep a bounded expansion of each fingerprint so simulated 80 GiB GPUs fit
#: on one B200; perf runs pass the model's real token_kv_bytes_per_layer.
DEFAULT_CELL_BYTES = 64
DEFAULT_MODEL_GROUPS = 64


def default_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return 0


class RequestRegistry:
    """Request id <-> int32 handle, shared by every store so a handle names the
    same request on a migration's source and destination."""

    def __init__(self) -> None:
        self._handle: dict = {}
        self._names: list = []
        self._rank: np.ndarray | None = None

    def handle(self, rid) -> int:
        h = self._handle.get(rid)
        if h is None:
            h = len(self._names)
            self._handle[rid] = h
            self._names.append(rid)
            self._rank = None
        return h

    def find(self, rid) -> int | None:
        return self._handle.get(rid)

    def name(self, h: int):
        return self._names[h]

    def rank(self) -> np.ndarray:
        """rank[h] = position of request h in sorted(request ids) (migrator.py:124)."""
        if self._rank is None or len(self._rank) != len(self._names):
            order = sorted(range(len(self._names)), key=lambda i: self._names[i])
            r = np.empty(len(order), dtype=np.int32)
            r[order] = np.arange(len(order), dtype=np.int32)
            self._rank = r
        return self._rank


REGISTRY = RequestRegistry()


@dataclass(frozen=True)
class StackedSlot:
    block_id: int
    layer_group: int
    offset: int
    checksum: int


class BlockView:
    """Read-only view of one physical block (PhysicalBlock, kvstore.py:47-61)."""

    __slots__ = ("_store", "block_id", "address", "capacity_tokens", "_owner", "slot")

    def __init__(self, store: "KvStore", block_id: int, owner: int, slot: int) -> None:
        self._store = store
        self.block_id = block_id
        self.address = store._address(block_id)
        self.capacity_tokens = store.tokens_per_block
        self._owner = owner
        self.slot = slot

    @property
    def owner(self):
        return None if self._owner < 0 else self._store._registry.name(self._owner)

    @property
    def state(self) -> str:
        return "live" if self._owner >= 0 else "free"

    def occupied_tokens(self) -> int:
        out = C.c_int64()
        _check(N.lib().pl_store_block_occupied(self._store._h, self.block_id, C.byref(out)))
        return out.value

    @property
    def cells(self) -> dict[int, dict[int, int]]:
        return self._store._block_cells(self.block_id, self.slot)

    def __repr__(self) -> str:
        return f"BlockView(id={self.block_id}, slot={self.slot}, {self.state})"


class TableView:
    """BlockTable view (kvstore.py:72-85): ``chain`` and ``written`` of one request."""

    def __init__(self, store: "KvStore", handle: int) -> None:
        self._store = store
        self._h = handle

    @property
    def written(self) -> dict[int, int]:
        return self._store._written(self._h)

    @property
    def chain(self) -> list[BlockView]:
        s = self._store
        ids = s._chain_ids(self._h)
        slots = s._chain_slots(self._h)
        return [BlockView(s, int(i), self._h, int(sl)) for i, sl in zip(ids, slots)]

    def addresses(self, group: int, tokens_per_block: int) -> list[int]:
        n = ceil(self.written.get(group, 0) / tokens_per_block)
        return [self._store._address(int(b)) for b in self._store._chain_ids(self._h)[:n]]


class TablesView:
    """Mapping request id -> TableView in dict insertion order (KvStore.tables)."""

    def __init__(self, store: "KvStore") -> None:
        self._store = store

    def _handles(self) -> list[int]:
        s = self._store
        n = C.c_int64()
        _check(N.lib().pl_store_tables(s._h, None, 0, C.byref(n)))
        buf = np.empty(max(n.value, 1), dtype=np.int32)
        _check(N.lib().pl_store_tables(s._h, N.ptr(buf), len(buf), C.byref(n)))
        return [int(x) for x in buf[: n.value]]

    def __contains__(self, rid) -> bool:
        h = self._store._registry.find(rid)
        return h is not None and self._store._has_table(h)

    def __getitem__(self, rid) -> TableView:
        h = self._store._registry.find(rid)
        if h is None or not self._store._has_table(h):
            raise KeyError(rid)
        return TableView(self._store, h)

    def get(self, rid, default=None):
        return self[rid] if rid in self else default

    def __iter__(self) -> Iterator:
        names = self._store._registry
        return iter([names.name(h) for h in self._handles()])

    def keys(self):
        return list(iter(self))

    def values(self):
        return [TableView(self._store, h) for h in self._handles()]

    def items(self):
        names = self._store._registry
        return [(names.name(h), TableView(self._store, h)) for h in self._handles()]

    def __len__(self) -> int:
        return self._store._info().n_tables

    def __bool__(self) -> bool:
        return len(self) > 0


class ResidentGroups(set):
    """The mutable ``resident_groups`` set; in-place edits (coordinator.py:205-206)
    map or release the group's device pool."""

    def __init__(self, store: "KvStore", groups: Iterable[int]) -> None:
        super().__init__(groups)
        self._store = store

    def _sync(self) -> None:
        self._store._sync_resident(set(self))

    def _wrap(name):  # noqa: N805
        base = getattr(set, name)

        def method(self, *args):
            out = base(self, *args)
            self._sync()
            return self if name.startswith("__i") else out

        method.__name__ = name
        return method

    for _n in ("add", "discard", "remove", "update", "difference_update",
               "intersection_update", "symmetric_difference_update", "clear", "pop",
               "__ior__", "__isub__", "__iand__", "__ixor__"):
        locals()[_n] = _wrap(_n)
    del _n, _wrap


class KvStore:
    """Block-granular, layer-stacked paged KV cache of one GPU (kvstore.py:88-360)."""

    def __init__(self, gpu_id: int, stacking_factor: int, tokens_per_block: int,
                 capacity_blocks: int, resident_groups: Iterable[int] = (), *,
                 num_groups: int | None = None, cell_bytes: int | None = None,
                 device: int | None = None, chunk_bytes: int = 0,
                 registry: RequestRegistry | None = None) -> None:
        if tokens_per_block <= 0:
            raise ValueError("tokens_per_block must be positive")
        groups = sorted(set(resident_groups))
        if num_groups is None:
            num_groups = max(DEFAULT_MODEL_GROUPS, (groups[-1] + 1) if groups else 0)
        self.gpu_id = gpu_id
        self.stacking_factor = stacking_factor
        self.tokens_per_block = tokens_per_block
        self.num_groups = num_groups
        self.cell_bytes = int(cell_bytes or DEFAULT_CELL_BYTES)
        self.device = default_device() if device is None else device
        self._registry = registry or REGISTRY
        self._h = None
        lib = N.lib()
        h = C.c_void_p()
        g = N.as_i32(groups) if groups else np.zeros(1, np.int32)
        _check(lib.pl_store_create(self.device, gpu_id, stacking_factor, tokens_per_block,
                                   self.cell_bytes, num_groups, capacity_blocks, N.ptr(g),
                                   len(groups), chunk_bytes, C.byref(h)))
        self._h = h
        self._resident = ResidentGroups(self, groups)
        self.tables = TablesView(self)

    def __del__(self) -> None:
        self.close()

    def close(self) -> None:
        """Destroy the native store now (device pools return to the driver once the
        reclaimer thread has unmapped them; the destructor joins it)."""
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.pl_store_destroy(h)
            self._h = None

    # -- helpers -------------------------------------------------------------------------
    def _info(self) -> N.StoreInfo:
        info = N.StoreInfo()
        _check(N.lib().pl_store_get_info(self._h, C.byref(info)))
        return info

    def _address(self, block_id: int) -> int:
        return (self.gpu_id << 44) | (block_id << 21)

    def _handle(self, rid) -> int:
        return self._registry.handle(rid)

    def _has_table(self, h: int) -> bool:
        out = C.c_int()
        _check(N.lib().pl_store_has_table(self._h, h, C.byref(out)))
        return bool(out.value)

    def _chain_ids(self, h: int) -> np.ndarray:
        n = C.c_int64()
        _check(N.lib().pl_store_chain(self._h, h, None, 0, C.byref(n)))
        buf = np.empty(max(n.value, 1), dtype=np.int64)
        _check(N.lib().pl_store_chain(self._h, h, N.ptr(buf), len(buf), C.byref(n)))
        return buf[: n.value]

    def _chain_slots(self, h: int) -> np.ndarray:
        n = C.c_int64()
        _check(N.lib().pl_store_chain_slots(self._h, h, None, 0, C.byref(n)))
        buf = np.empty(max(n.value, 1), dtype=np.int32)
        _check(N.lib().pl_store_chain_slots(self._h, h, N.ptr(buf), len(buf), C.byref(n)))
        return buf[: n.value]

    _WCAP = 256
    _wg = (C.c_int32 * _WCAP)()
    _wc = (C.c_int64 * _WCAP)()
    _wn = C.c_int()

    def _written(self, h: int) -> dict[int, int]:
        """The request's written counts per group, in dict insertion order (one C call;
        preallocated buffers: this is on the parity-mode control plane's hot path)."""
        cls = KvStore
        _check(N.lib().pl_store_written(self._h, h, cls._wg, cls._wc, cls._WCAP, C.byref(cls._wn)))
        n = cls._wn.value
        if n > cls._WCAP:
            gs = (C.c_int32 * n)()
            cs = (C.c_int64 * n)()
            _check(N.lib().pl_store_written(self._h, h, gs, cs, n, C.byref(cls._wn)))
            return dict(zip(gs, cs))
        return dict(zip(cls._wg[:n], cls._wc[:n]))

    def written(self, request_id, group: int) -> int:
        """Fast path for ``tables[rid].written.get(group, 0)``."""
        h = self._registry.find(request_id)
        if h is None:
            return 0
        return self._written(h).get(group, 0)

    def written_all(self, request_id) -> dict[int, int]:
        """``tables[rid].written`` as a plain dict (empty when the request has no table)."""
        h = self._registry.find(request_id)
        return {} if h is None else self._written(h)

    def _sync_resident(self, wanted: set[int]) -> None:
        cur = set(self._resident_native())
        add = sorted(wanted - cur)
        rem = sorted(cur - wanted)
        if add:
            a = N.as_i32(add)
            _check(N.lib().pl_store_add_groups(self._h, N.ptr(a), len(add)))
        if rem:
            r = N.as_i32(rem)
            _check(N.lib().pl_store_remove_groups(self._h, N.ptr(r), len(rem)))

    def _resident_native(self) -> list[int]:
        buf = np.empty(self.num_groups, dtype=np.int32)
        n = C.c_int()
        _check(N.lib().pl_store_resident(self._h, N.ptr(buf), len(buf), C.byref(n)))
        return [int(x) for x in buf[: n.value]]

    def _read_fps(self, group: int, slots: np.ndarray) -> np.ndarray:
        out = np.empty((len(slots), self.tokens_per_block), dtype=np.uint64)
        if len(slots):
            sl = N.as_i32(slots)
            _check(N.lib().pl_store_read_fps(self._h, group, N.ptr(sl), len(sl), N.ptr(out)))
        return out

    def _occupancy(self, block_id: int, group: int) -> int:
        words = np.zeros(16, dtype=np.uint64)
        n = C.c_int()
        _check(N.lib().pl_store_block_occupancy(self._h, block_id, group, N.ptr(words), 16,
                                                C.byref(n)))
        if n.value > 16:
            words = np.zeros(n.value, dtype=np.uint64)
            _check(N.lib().pl_store_block_occupancy(self._h, block_id, group, N.ptr(words),
                                                    n.value, C.byref(n)))
        mask = 0
        for i in range(n.value):
            mask |= int(words[i]) << (64 * i)
        return mask

    def _block_cells(self, block_id: int, slot: int) -> dict[int, dict[int, int]]:
        cells: dict[int, dict[int, int]] = {}
        for g in range(self.num_groups):
            mask = self._occupancy(block_id, g)
            if not mask:
                continue
            fps = self._read_fps(g, np.array([slot], dtype=np.int32))[0]
            cells[g] = {o: int(fps[o]) for o in range(self.tokens_per_block) if (mask >> o) & 1}
        return cells

    # -- accounting ----------------------------------------------------------------------
    @property
    def resident_groups(self) -> ResidentGroups:
        return self._resident

    @resident_groups.setter
    def resident_groups(self, value: Iterable[int]) -> None:
        wanted = set(value)
        if value is not self._resident:
            set.clear(self._resident)
            set.update(self._resident, wanted)
        self._sync_resident(wanted)

    @property
    def capacity_blocks(self) -> int:
        return self._info().capacity_blocks

    @property
    def used_blocks(self) -> int:
        return self._info().used_blocks

    @property
    def free_blocks(self) -> int:
        return self._info().free_blocks

    @property
    def occupied_cells(self) -> int:
        return self._info().occupied_cells

    @property
    def blocks(self) -> list[BlockView]:
        n = C.c_int64()
        _check(N.lib().pl_store_blocks(self._h, None, None, None, 0, C.byref(n)))
        m = max(n.value, 1)
        ids = np.empty(m, dtype=np.int64)
        owner = np.empty(m, dtype=np.int32)
        slot = np.empty(m, dtype=np.int32)
        _check(N.lib().pl_store_blocks(self._h, N.ptr(ids), N.ptr(owner), N.ptr(slot), m,
                                       C.byref(n)))
        return [BlockView(self, int(ids[i]), int(owner[i]), int(slot[i])) for i in range(n.value)]

    def chain_len(self, request_id) -> int:
        h = self._registry.find(request_id)
        return 0 if h is None else len(self._chain_ids(h))

    def blocks_needed(self, request_id, extra_tokens: int) -> int:
        h = self._registry.find(request_id)
        if h is None:
            return max(0, ceil(extra_tokens / self.tokens_per_block))
        out = C.c_int64()
        _check(N.lib().pl_store_blocks_needed(self._h, h, extra_tokens, C.byref(out)))
        return out.value

    # -- operations (kvstore.py:163-322) ---------------------------------------------------
    def append(self, request_id, layer_group: int, n_tokens: int,
               payload_checksums: Sequence[int]) -> list[StackedSlot]:
        if n_tokens != len(payload_checksums):
            raise ValueError("one checksum per token required")
        if n_tokens == 0:
            return []
        h = self._handle(request_id)
        pay = N.as_u64([int(x) for x in payload_checksums])
        _check(N.lib().pl_store_append(self._h, h, layer_group, n_tokens, N.PL_PAYLOAD_EXPLICIT,
                                       N.ptr(pay), 0, None, 0))
        s = self.tokens_per_block
        end = self._written(h)[layer_group]
        start = end - n_tokens
        chain = self._chain_ids(h)
        return [StackedSlot(int(chain[(start + i) // s]), layer_group, (start + i) % s,
                            int(payload_checksums[i])) for i in range(n_tokens)]

    def append_seeded(self, request_id, layer_group: int, n_tokens: int, seed: int,
                      kv_dev: int | None = None, mark: bool = False) -> None:
        """Engine path: payload = engine.py:252-261 fingerprints of ``seed``, computed
        on device; ``kv_dev`` optionally supplies real KV bytes [n][k][cell_bytes]."""
        if n_tokens <= 0:
            return
        h = self._handle(request_id)
        if kv_dev is not None:
            self.wait_for_caller_stream()
        _check(N.lib().pl_store_append(self._h, h, layer_group, n_tokens, N.PL_PAYLOAD_SEED,
                                       None, seed, kv_dev, 1 if mark else 0))

    def stream_ptr(self) -> int:
        """The cudaStream_t this store's work is enqueued on."""
        out = C.c_void_p()
        _check(N.lib().pl_store_stream(self._h, C.byref(out)))
        return out.value or 0

    def wait_for_caller_stream(self, stream_ptr: int | None = None) -> None:
        """Order the store's stream after the caller's (default: torch's current stream),
        so device buffers the caller just produced (kv_dev) are complete when K1 reads."""
        if stream_ptr is None:
            try:
                import torch
                stream_ptr = torch.cuda.current_stream(self.device).cuda_stream
            except Exception:  # pragma: no cover - torch is plumbing only
                stream_ptr = 0
        _check(N.lib().pl_store_wait_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def append_groups_seeded(self, request_id, groups: list[int], n_tokens: int,
                             seeds: list[int], start: int | None = None,
                             mark: bool = False) -> tuple[int, bool]:
        """Engine path (engine.py:392-400): append n_tokens to each group in order with
        fingerprints of positions start.. (default: each group's written prefix), one K1
        launch.  Stops at the first overflow; returns (groups done, overflowed).  With
        ``mark`` the same launch sets the dirty bits of every active migration patch
        streaming those groups (the DirtyBitmap.mark of migrator.py:190-197)."""
        if not groups or n_tokens <= 0:
            return 0, False
        h = self._handle(request_id)
        m = len(groups)
        reqs = np.full(m, h, dtype=np.int32)
        gs = N.as_i32(groups)
        counts = np.full(m, n_tokens, dtype=np.int64)
        sd = N.as_u64(seeds)
        fs = None if start is None else np.full(m, start, dtype=np.int64)
        done = C.c_int()
        rc = N.lib().pl_store_append_batch(self._h, m, N.ptr(reqs), N.ptr(gs), N.ptr(counts),
                                           N.ptr(sd), N.ptr(fs), None, 1 if mark else 0,
                                           C.byref(done), None, 0)
        if rc == N.PL_E_KV_OVERFLOW:
            return done.value, True
        _check(rc)
        return done.value, False

    def write_slots(self, request_id, layer_group: int,
                    items: Sequence[tuple[int, int]]) -> None:
        if not items:
            return
        h = self._handle(request_id)
        pos = N.as_i64([int(p) for p, _ in items])
        pay = N.as_u64([int(c) for _, c in items])
        _check(N.lib().pl_store_write_slots(self._h, h, layer_group, len(items), N.ptr(pos),
                                            N.ptr(pay)))

    def lookup(self, request_id, layer: int, token_idx: int) -> tuple[int, int]:
        h = self._registry.find(request_id)
        if h is None:
            raise UnknownSlot(f"{request_id} layer {layer} token {token_idx}")
        addr = C.c_uint64()
        off = C.c_int64()
        rc = N.lib().pl_store_lookup(self._h, h, layer, token_idx, C.byref(addr), C.byref(off))
        if rc == N.PL_E_UNKNOWN_SLOT:
            raise UnknownSlot(f"{request_id} layer {layer} token {token_idx}")
        _check(rc)
        return addr.value, off.value

    def read_checksum(self, request_id, layer_group: int, token_idx: int) -> int:
        h = self._registry.find(request_id)
        if h is None:
            raise UnknownSlot(f"{request_id} group {layer_group} token {token_idx}")
        out = C.c_uint64()
        rc = N.lib().pl_store_read_checksum(self._h, h, layer_group, token_idx, C.byref(out))
        if rc == N.PL_E_UNKNOWN_SLOT:
            raise UnknownSlot(f"{request_id} group {layer_group} token {token_idx}")
        _check(rc)
        return out.value

    def read_cell(self, request_id, layer_group: int, token_idx: int, layer_in_group: int,
                  nbytes: int | None = None) -> bytes:
        """Raw KV bytes of one (token, layer) cell (parity checks)."""
        h = self._registry.find(request_id)
        if h is None:
            raise UnknownSlot(str(request_id))
        n = nbytes or self.cell_bytes
        buf = np.empty(n, dtype=np.uint8)
        _check(N.lib().pl_store_read_cell(self._h, h, layer_group, token_idx, layer_in_group,
                                          N.ptr(buf), n))
        return buf.tobytes()

    def verify_cells(self, seeds: dict | None = None) -> dict[str, int]:
        """Every live cell on the device (csrc/verify.cu): all k layer cells must be the
        parity expansion of the cell's fingerprint; with ``seeds`` ({(request_id, group):
        seed}), each fingerprint must also be PipelineEngine._payloads' value for its
        position (engine.py:252-261).  Returns the kernel's counters."""
        arr, n = None, 0
        if seeds:
            n = max(self._registry.handle(r) for r, _ in seeds) + 1
            arr = np.full((n, self.num_groups), np.iinfo(np.uint64).max, dtype=np.uint64)
            for (r, g), sd in seeds.items():
                arr[self._registry.handle(r), g] = sd
        out = np.zeros(4, dtype=np.int64)
        _check(N.lib().pl_store_verify(self._h, N.ptr(arr), n, N.ptr(out)))
        return {"cells": int(out[0]), "bad_bytes": int(out[1]), "bad_fingerprints": int(out[2]),
                "first_bad": int(out[3])}

    def compare_cells(self, other: "KvStore", groups: Iterable[int],
                      request_ids: Iterable | None = None) -> dict[str, int]:
        """Byte-for-byte comparison with another store on the same device: every written
        position (the shorter prefix of the two) of every (request, group), fingerprint and
        k cells, each side through its own block table.  Default requests: all of this
        store's."""
        rids = list(self.tables) if request_ids is None else list(request_ids)
        groups = list(groups)
        hs = N.as_i32([self._registry.handle(r) for r in rids] or [0])
        gs = N.as_i32(groups or [0])
        out = np.zeros(4, dtype=np.int64)
        _check(N.lib().pl_store_compare(self._h, other._h, N.ptr(gs), len(groups),
                                        N.ptr(hs), len(rids), N.ptr(out)))
        return {"cells": int(out[0]), "bad_positions": int(out[1]), "missing": int(out[2]),
                "length_mismatch": int(out[3])}

    def compact(self) -> int:
        out = C.c_int64()
        _check(N.lib().pl_store_compact(self._h, C.byref(out)))
        return out.value

    def resize(self, new_capacity: int) -> None:
        _check(N.lib().pl_store_resize(self._h, new_capacity))

    def last_resize_stats(self) -> dict[str, int]:
        out = np.zeros(4, dtype=np.int64)
        _check(N.lib().pl_store_last_resize_stats(self._h, N.ptr(out)))
        return {"relocated_blocks": int(out[0]), "table_entries_remapped": int(out[1]),
                "bytes_mapped": int(out[2]), "bytes_unmapped": int(out[3])}

    def vmm_stats(self) -> dict[str, int]:
        """Physical-memory bookkeeping of the pools (vmm.cu): chunks re-taken from a
        retired but still mapped tail, re-mapped from the reclaimer's cache, freshly
        created, and bytes not yet returned to the driver."""
        out = np.zeros(4, dtype=np.int64)
        _check(N.lib().pl_store_vmm_stats(self._h, N.ptr(out)))
        return {"tail_reused_chunks": int(out[0]), "cache_reused_chunks": int(out[1]),
                "created_chunks": int(out[2]), "pending_reclaim_bytes": int(out[3])}

    def staging_stats(self) -> dict[str, int]:
        """The H2D staging ring behind every upload (store.cu stage_span): capacity, growths,
        spans retired with a host wait, host ns spent acquiring spans (total, longest),
        outgrown rings not yet freed (they are freed at sync(), a host sync point)."""
        out = np.zeros(6, dtype=np.int64)
        _check(N.lib().pl_store_staging_stats(self._h, N.ptr(out)))
        return dict(zip(("ring_bytes", "outgrows", "retire_waits", "wait_ns", "span_max_ns",
                         "old_rings"), (int(x) for x in out)))

    def prepare_grow(self, new_capacity: int, groups: Iterable[int]) -> int:
        """Create, on the reclaimer thread, the physical chunks a planned
        resize(new_capacity) with `groups` resident will need; returns chunks requested."""
        g = N.as_i32(sorted(groups))
        out = C.c_int64()
        _check(N.lib().pl_store_prepare_grow(self._h, new_capacity, N.ptr(g), len(g),
                                             C.byref(out)))
        return out.value

    def prepare_wait(self) -> float:
        out = C.c_double()
        _check(N.lib().pl_store_prepare_wait(self._h, C.byref(out)))
        return out.value

    def reclaim(self) -> float:
        """Finish every deferred unmap/release now; returns the wait in ms."""
        out = C.c_double()
        _check(N.lib().pl_store_reclaim(self._h, C.byref(out)))
        return out.value

    def drop_layer_groups(self, layer_groups: Iterable[int]) -> int:
        groups = sorted(set(layer_groups))
        g = N.as_i32(groups) if groups else np.zeros(1, np.int32)
        out = C.c_int64()
        _check(N.lib().pl_store_drop_groups(self._h, N.ptr(g), len(groups), C.byref(out)))
        set.difference_update(self._resident, groups)
        return out.value

    def free_request(self, request_id) -> dict[int, tuple[int, int]]:
        h = self._registry.find(request_id)
        if h is None:
            return {}
        cap = 64
        stats = np.zeros(3 * cap, dtype=np.int64)
        n = C.c_int()
        _check(N.lib().pl_store_free_request(self._h, h, N.ptr(stats), cap, C.byref(n)))
        return {int(stats[3 * i]): (int(stats[3 * i + 1]), int(stats[3 * i + 2]))
                for i in range(min(n.value, cap))}

    def free_requests(self, request_ids: Iterable) -> None:
        """free_request for many requests at once (one C-ABI call; no per-group stats)."""
        hs = [h for h in (self._registry.find(r) for r in request_ids) if h is not None]
        if hs:
            arr = N.as_i32(hs)
            _check(N.lib().pl_store_free_requests(self._h, len(hs), N.ptr(arr)))

    def effective_utilization(self) -> float:
        out = C.c_double()
        _check(N.lib().pl_store_utilization(self._h, C.byref(out)))
        return out.value

    def snapshot_group(self, layer_group: int) -> dict[object, tuple[int, ...]]:
        out: dict[object, tuple[int, ...]] = {}
        names = self._registry
        for rid in sorted(self.tables):
            h = names.find(rid)
            w = self._written(h).get(layer_group, 0)
            if w == 0:
                continue
            slots = self._chain_slots(h)[: ceil(w / self.tokens_per_block)]
            fps = self._read_fps(layer_group, slots).reshape(-1)[:w]
            out[rid] = tuple(int(x) for x in fps)
        return out

    def state_digest(self) -> tuple:
        tables = []
        names = self._registry
        for rid in sorted(self.tables):
            h = names.find(rid)
            ids = self._chain_ids(h)
            slots = self._chain_slots(h)
            per_block: list[dict[int, dict[int, int]]] = [dict() for _ in ids]
            for g in range(self.num_groups):
                masks = [self._occupancy(int(b), g) for b in ids]
                if not any(masks):
                    continue
                fps = self._read_fps(g, slots)
                for i, m in enumerate(masks):
                    if m:
                        per_block[i][g] = {o: int(fps[i][o]) for o in range(self.tokens_per_block)
                                           if (m >> o) & 1}
            tables.append((
                rid,
                tuple(sorted(self._written(h).items())),
                tuple(tuple(sorted((g, tuple(sorted(c.items()))) for g, c in cells.items()))
                      for cells in per_block),
            ))
        return (self.capacity_blocks, self.used_blocks, tuple(sorted(self.resident_groups)),
                tuple(tables))

    # -- device views ----------------------------------------------------------------------
    def group_base(self, group: int) -> int:
        out = C.c_uint64()
        _check(N.lib().pl_store_group_base(self._h, group, C.byref(out)))
        return out.value

    def table_device(self) -> tuple[int, int]:
        p = C.c_uint64()
        stride = C.c_int64()
        _check(N.lib().pl_store_table_dev(self._h, C.byref(p), C.byref(stride)))
        return p.value, stride.value

    def sync(self) -> None:
        _check(N.lib().pl_store_sync(self._h))

    def info(self) -> dict[str, int]:
        i = self._info()
        return {name: getattr(i, name) for name, _ in N.StoreInfo._fields_}


def default_cell_bytes(model: ModelSpec) -> int:
    """Parity runs store min(token_kv_bytes_per_layer, DEFAULT_CELL_BYTES) bytes per
    cell (a prefix of the deterministic expansion); rounded to 16 B."""
    b = min(model.token_kv_bytes_per_layer, DEFAULT_CELL_BYTES)
    return max(16, (b + 15) // 16 * 16)


def kv_init(gpu: GpuSpec, model: ModelSpec, capacity_blocks: int,
            resident_groups: Iterable[int] = (), weight_bytes: int = 0, *,
            cell_bytes: int | None = None, device: int | None = None,
            registry: RequestRegistry | None = None, chunk_bytes: int = 0) -> KvStore:
    """Empty store after the simulated memory check (kvstore.py:363-373)."""
    groups = set(resident_groups)
    kv_bytes = capacity_blocks * gpu.alloc_granularity * max(1, len(groups))
    if kv_bytes + weight_bytes > gpu.mem_total:
        raise InsufficientMemory(
            f"gpu {gpu.id}: {kv_bytes + weight_bytes} B exceeds {gpu.mem_total} B")
    # the model's group count from the fields every ModelSpec has (the reference's own
    # ModelSpec has no num_groups: a maintainer's shim hands it to this kv_init unchanged)
    n_groups = -(-model.num_layers // model.stacking_factor)
    return KvStore(gpu.id, model.stacking_factor, model.tokens_per_block(gpu), capacity_blocks,
                   groups, num_groups=max(n_groups, DEFAULT_MODEL_GROUPS),
                   cell_bytes=cell_bytes or default_cell_bytes(model), device=device,
                   registry=registry, chunk_bytes=chunk_bytes)
