"""ctypes binding of libpipelive.so (include/pipelive.h).

The product path has no CPU fallback: importing the data-plane classes works
anywhere (so the CPU test-suite can check the ABI), but the first call that
needs the library raises NativeUnavailable unless libpipelive.so is built and
a CUDA device is visible.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PIPELIVE_LIB", _HERE / "libpipelive.so"))

PL_OK = 0
PL_E_KV_OVERFLOW = -1
PL_E_CAPACITY_BELOW_LIVE = -2
PL_E_UNKNOWN_SLOT = -3
PL_E_UNKNOWN_LAYER_GROUP = -4
PL_E_INSUFFICIENT_MEMORY = -5
PL_E_INVALID = -6
PL_E_CUDA = -7
PL_E_STATE = -8

PL_PAYLOAD_EXPLICIT = 0
PL_PAYLOAD_SEED = 1


class NativeUnavailable(RuntimeError):
    """libpipelive.so is missing or no CUDA device is visible (no CPU fallback exists)."""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str) -> None:
        super().__init__(msg)
        self.code = code


class StoreInfo(C.Structure):
    _fields_ = [(name, C.c_int64) for name in (
        "capacity_blocks", "used_blocks", "free_blocks", "occupied_cells", "n_resident",
        "tokens_per_block", "stacking_factor", "cell_bytes", "unit_bytes", "fp_header_bytes",
        "mapped_bytes", "table_max_chain", "table_max_reqs", "n_tables")]


i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P = C.POINTER

# (name, restype, argtypes) -- every symbol declared in include/pipelive.h
SIGNATURES = [
    ("pl_last_error", C.c_char_p, []),
    ("pl_abi_version", C.c_int, []),
    ("pl_device_count", C.c_int, [P(C.c_int)]),
    ("pl_store_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, i64, C.c_int, i64, vp,
                                  C.c_int, i64, P(vp)]),
    ("pl_store_destroy", C.c_int, [vp]),
    ("pl_store_set_stream", C.c_int, [vp, vp]),
    ("pl_store_wait_stream", C.c_int, [vp, vp]),
    ("pl_store_get_info", C.c_int, [vp, P(StoreInfo)]),
    ("pl_store_add_groups", C.c_int, [vp, vp, C.c_int]),
    ("pl_store_remove_groups", C.c_int, [vp, vp, C.c_int]),
    ("pl_store_resident", C.c_int, [vp, vp, C.c_int, P(C.c_int)]),
    ("pl_store_blocks_needed", C.c_int, [vp, i32, i64, P(i64)]),
    ("pl_store_chain", C.c_int, [vp, i32, vp, i64, P(i64)]),
    ("pl_store_chain_slots", C.c_int, [vp, i32, vp, i64, P(i64)]),
    ("pl_store_written", C.c_int, [vp, i32, vp, vp, C.c_int, P(C.c_int)]),
    ("pl_store_has_table", C.c_int, [vp, i32, P(C.c_int)]),
    ("pl_store_tables", C.c_int, [vp, vp, i64, P(i64)]),
    ("pl_store_blocks", C.c_int, [vp, vp, vp, vp, i64, P(i64)]),
    ("pl_store_block_occupied", C.c_int, [vp, i64, P(i64)]),
    ("pl_store_block_occupancy", C.c_int, [vp, i64, C.c_int, vp, C.c_int, P(C.c_int)]),
    ("pl_store_append", C.c_int, [vp, i32, C.c_int, i64, C.c_int, vp, u64, vp, C.c_int]),
    ("pl_store_append_batch", C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp, C.c_int,
                                        P(C.c_int), vp, C.c_int]),
    ("pl_store_append_batch_payloads", C.c_int, [vp, C.c_int, vp, vp, vp, vp, C.c_int, P(C.c_int)]),
    ("pl_store_write_slots", C.c_int, [vp, i32, C.c_int, i64, vp, vp]),
    ("pl_store_write_layer", C.c_int, [vp, C.c_int, C.c_int, vp, vp, C.c_int, vp, i64, vp]),
    ("pl_store_lookup", C.c_int, [vp, i32, C.c_int, i64, P(u64), P(i64)]),
    ("pl_store_read_checksum", C.c_int, [vp, i32, C.c_int, i64, P(u64)]),
    ("pl_store_read_fps", C.c_int, [vp, C.c_int, vp, i64, vp]),
    ("pl_store_read_cell", C.c_int, [vp, i32, C.c_int, i64, C.c_int, vp, i64]),
    ("pl_store_verify", C.c_int, [vp, vp, i64, vp]),
    ("pl_store_compare", C.c_int, [vp, vp, vp, C.c_int, vp, C.c_int, vp]),
    ("pl_act_ring_create", C.c_int, [C.c_int, i64, C.c_int, P(vp)]),
    ("pl_act_ring_export", C.c_int, [vp, vp, i64, P(i64)]),
    ("pl_act_ring_open", C.c_int, [C.c_int, vp, i64, P(vp)]),
    ("pl_act_ring_destroy", C.c_int, [vp]),
    ("pl_act_send", C.c_int, [vp, vp, i64, vp]),
    ("pl_act_recv", C.c_int, [vp, vp, i64, vp]),
    ("pl_mailbox_create", C.c_int, [C.c_int, i64, C.c_int, P(vp)]),
    ("pl_mailbox_export", C.c_int, [vp, vp, i64, P(i64)]),
    ("pl_mailbox_open", C.c_int, [C.c_int, vp, i64, P(vp)]),
    ("pl_mailbox_destroy", C.c_int, [vp]),
    ("pl_mailbox_base", C.c_int, [vp, P(vp), P(i64)]),
    ("pl_mailbox_post", C.c_int, [vp, i64, u64]),
    ("pl_mailbox_wait", C.c_int, [vp, i64, u64, i64, P(u64)]),
    ("pl_mailbox_record", C.c_int, [vp, C.c_int, vp]),
    ("pl_mailbox_stream_wait", C.c_int, [vp, C.c_int, vp]),
    ("pl_pair_send_rows", C.c_int, [vp, vp, vp, i64, u64, P(i64), P(i64), P(i64)]),
    ("pl_pair_serve_rows", C.c_int, [vp, vp, vp, C.c_int, u64, i64, vp, P(C.c_int), P(i64)]),
    ("pl_pair_finish", C.c_int, [vp, vp, vp, u64, i64, C.c_int, P(C.c_int), P(C.c_int),
                                 P(i64)]),
    ("pl_pair_serve_ack", C.c_int, [vp, vp, u64, i64]),
    ("pl_store_export_versions", C.c_int, [vp, vp, C.c_int, vp]),
    ("pl_exact_gemv", C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp]),
    ("pl_exact_rmsnorm", C.c_int, [vp, vp, vp, C.c_int, C.c_int, dbl, vp]),
    ("pl_exact_rope_pack", C.c_int, [vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int,
                                     C.c_int, vp]),
    ("pl_exact_silu_mul", C.c_int, [vp, vp, vp, i64, vp]),
    ("pl_exact_attn_decode", C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, C.c_int,
                                       C.c_int, C.c_int, dbl, C.c_int, vp]),
    ("pl_store_compact", C.c_int, [vp, P(i64)]),
    ("pl_store_resize", C.c_int, [vp, i64]),
    ("pl_store_drop_groups", C.c_int, [vp, vp, C.c_int, P(i64)]),
    ("pl_store_free_request", C.c_int, [vp, i32, vp, C.c_int, P(C.c_int)]),
    ("pl_store_free_requests", C.c_int, [vp, C.c_int, vp]),
    ("pl_store_utilization", C.c_int, [vp, P(dbl)]),
    ("pl_store_last_resize_stats", C.c_int, [vp, vp]),
    ("pl_store_vmm_stats", C.c_int, [vp, vp]),
    ("pl_store_staging_stats", C.c_int, [vp, vp]),
    ("pl_store_reclaim", C.c_int, [vp, P(dbl)]),
    ("pl_store_prepare_grow", C.c_int, [vp, i64, vp, C.c_int, P(i64)]),
    ("pl_store_prepare_wait", C.c_int, [vp, P(dbl)]),
    ("pl_store_group_base", C.c_int, [vp, C.c_int, P(u64)]),
    ("pl_store_table_dev", C.c_int, [vp, P(u64), P(i64)]),
    ("pl_store_flush", C.c_int, [vp]),
    ("pl_store_sync", C.c_int, [vp]),
    ("pl_patch_create", C.c_int, [vp, vp, vp, C.c_int, P(vp)]),
    ("pl_patch_destroy", C.c_int, [vp]),
    ("pl_patch_set_active", C.c_int, [vp, C.c_int]),
    ("pl_patch_mark", C.c_int, [vp, i32, C.c_int, i64, i64]),
    ("pl_patch_mark_batch", C.c_int, [vp, C.c_int, vp, vp, vp, vp]),
    ("pl_patch_set_stream", C.c_int, [vp, vp]),
    ("pl_patch_seed", C.c_int, [vp, P(i64)]),
    ("pl_patch_discard_request", C.c_int, [vp, i32, P(i64)]),
    ("pl_patch_dirty_keys", C.c_int, [vp, P(i64)]),
    ("pl_patch_drain", C.c_int, [vp, P(i64), P(i64)]),
    ("pl_patch_drained_keys", C.c_int, [vp, vp, vp, vp, i64, P(i64)]),
    ("pl_patch_apply", C.c_int, [vp, vp, vp, i64, vp, i64]),
    ("pl_patch_push", C.c_int, [vp, vp, vp, i64, P(i64), P(i64)]),
    ("pl_patch_last_push_stats", C.c_int, [vp, vp]),
    ("pl_patch_stream", C.c_int, [vp, P(vp)]),
    ("pl_store_stream", C.c_int, [vp, P(vp)]),
    ("pl_patch_device_dirty_count", C.c_int, [vp, P(i64)]),
    ("pl_patch_device_drained", C.c_int, [vp, P(i64)]),
    ("pl_patch_device_drained_async", C.c_int, [vp, vp]),
    ("pl_store_layout", C.c_int, [vp, vp]),
    ("pl_store_export_group", C.c_int, [vp, C.c_int, vp, C.c_int, P(C.c_int), P(i64)]),
    ("pl_store_export_table", C.c_int, [vp, vp, P(i64), P(i64)]),
    ("pl_store_table_version", C.c_int, [vp, P(u64), P(i64), P(i64)]),
    ("pl_store_reserve_rows", C.c_int, [vp, i64, vp, vp, vp, vp, P(i64)]),
    ("pl_remote_create", C.c_int, [C.c_int, C.c_int, C.c_int, i64, i64, i64, C.c_int, P(vp)]),
    ("pl_remote_destroy", C.c_int, [vp]),
    ("pl_remote_destroy_after", C.c_int, [vp, vp]),
    ("pl_remote_import_group", C.c_int, [vp, C.c_int, vp, C.c_int, i64]),
    ("pl_remote_drop_group", C.c_int, [vp, C.c_int]),
    ("pl_remote_set_table", C.c_int, [vp, vp, i64, i64]),
    ("pl_patch_drain_rows", C.c_int, [vp, vp, i64, P(i64), P(i64), P(i64)]),
    ("pl_patch_rows", C.c_int, [vp, vp, vp, vp, vp, i64]),
    ("pl_patch_push_remote", C.c_int, [vp, vp, i64]),
    ("pl_paged_attn_decode", C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_float, C.c_int, vp]),
    ("pl_paged_attn_decode_raw", C.c_int, [vp, i64, i64, C.c_int, C.c_int, C.c_int, vp, vp, vp,
                                           C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_float, C.c_int, vp]),
    ("pl_launch_count", i64, []),
    ("pl_timing_enable", C.c_int, [C.c_int]),
    ("pl_timing_read", C.c_int, [C.c_char_p, P(dbl), P(i64)]),
    ("pl_timing_reset", C.c_int, []),
]

_lib = None
_device_ok = False


def load_library(path: Path | None = None, require_device: bool = True):
    """Load and type the C-ABI; raise NativeUnavailable when it cannot run here."""
    global _lib, _device_ok
    if _lib is not None and path is None:
        if require_device and not _device_ok:
            _require_device(_lib)
            _device_ok = True
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    if require_device:
        _require_device(lib)
    return lib


def _require_device(lib) -> None:
    n = C.c_int(0)
    rc = lib.pl_device_count(C.byref(n))
    if rc != PL_OK or n.value <= 0:
        raise NativeUnavailable("no CUDA device visible: the pipelive data path is GPU-only "
                                "(no CPU fallback by design)")


def lib():
    if _device_ok:          # hot path: every ctypes call of the parity-mode control plane
        return _lib
    return load_library()


def check(rc: int) -> None:
    if rc != PL_OK:
        msg = _lib.pl_last_error().decode(errors="replace") if _lib is not None else ""
        raise NativeError(rc, msg)


def ptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


def as_i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def as_i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def as_u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


def launch_count() -> int:
    return int(lib().pl_launch_count())


def timing(kernel: str) -> tuple[float, int]:
    """(summed device ms, launches) of one instrumented kernel since the last reset."""
    ms = C.c_double()
    n = C.c_int64()
    check(lib().pl_timing_read(kernel.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value
