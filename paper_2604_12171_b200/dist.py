"""One process per GPU: the cross-process halves of the patch path and stage activations.

- ``Channel``: a Unix-domain stream socket between two local ranks.  It carries pickled
  control messages (a few KB per patch round) and, with SCM_RIGHTS, the POSIX fds of the
  destination's exported VMM pool chunks.  Both stages of a migrating pair are on one
  node (NVSwitch), so a local socket is enough; nothing here touches NCCL.
- ``RemoteStore``: the sender's view of the receiver's store (pools imported from the
  fds, block table opened from a CUDA IPC handle), used by the fused push kernel to
  write the receiver's cells directly (NVLink stores when the GPUs differ).
- ``PatchSender`` / ``PatchReceiver``: one migrating (src, dst) pair split across the two
  processes.  Per round (MigrationStream.pump -> _drain -> _send_patch ->
  PatchReceiver.receive, migrator.py:208-273, 93-132): sender drains rows + K3 ->
  receiver reserves the positions with the reference's block-id policy and publishes
  its table -> sender pushes (K4+K5) -> sender's stream is synchronised -> "applied".
- ``StageLink`` / ``ActRing``: stage-to-stage activations (engine.py:353-375,
  fabric.py:129-136, K7): by default device-to-device through a ring the receiving stage
  owns (csrc/act.cu: CUDA IPC buffers + interprocess events + a shared-memory mailbox);
  NCCL isend/irecv or gloo (host-staged, CPU tests) as alternatives.
"""

from __future__ import annotations

import ctypes as C
import os
import pickle
import socket
import struct
import time

import numpy as np

from . import _native as N
from .kvstore import KvStore, _check
from .perf import NativePatch

_HDR = struct.Struct("<QI")


class Channel:
    """Local socket between two processes; ``name`` is shared, one side is the server.

    ``Channel(name, server)`` blocks until connected.  Ranks that are server of one pair
    and client of another (a ring of pairs) use ``Channel.listen`` first, then
    ``Channel.connect``, then ``Listener.accept`` so no rank waits in accept while its
    own peer waits in accept too."""

    class Listener:
        def __init__(self, name: str, timeout: float) -> None:
            self.ls = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            self.ls.bind("\0pipelive-" + name)   # Linux abstract namespace: no file
            self.ls.listen(1)
            self.ls.settimeout(timeout)

        def accept(self) -> "Channel":
            sock, _ = self.ls.accept()
            self.ls.close()
            return Channel._wrap(sock)

    @classmethod
    def listen(cls, name: str, timeout: float = 120.0) -> "Channel.Listener":
        return cls.Listener(name, timeout)

    @classmethod
    def connect(cls, name: str, timeout: float = 120.0) -> "Channel":
        deadline = time.time() + timeout
        while True:
            s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            try:
                s.connect("\0pipelive-" + name)
                return cls._wrap(s)
            except OSError:
                s.close()
                if time.time() > deadline:
                    raise
                time.sleep(0.02)

    @classmethod
    def _wrap(cls, sock) -> "Channel":
        ch = cls.__new__(cls)
        sock.settimeout(None)
        ch.sock = sock
        return ch

    def __init__(self, name: str, server: bool, timeout: float = 120.0) -> None:
        ch = (Channel.listen(name, timeout).accept() if server
              else Channel.connect(name, timeout))
        self.sock = ch.sock

    MAX_FDS = 250   # SCM_RIGHTS carries at most 253 descriptors per message

    def send(self, obj, fds=()) -> None:
        data = pickle.dumps(obj)
        fds = list(fds)
        socket.send_fds(self.sock, [_HDR.pack(len(data), len(fds))], fds[: self.MAX_FDS])
        for i in range(self.MAX_FDS, len(fds), self.MAX_FDS):
            socket.send_fds(self.sock, [b"+"], fds[i:i + self.MAX_FDS])
        self.sock.sendall(data)

    def recv(self):
        hdr, fds, _, _ = socket.recv_fds(self.sock, _HDR.size, 4096)
        while len(hdr) < _HDR.size:
            more = self.sock.recv(_HDR.size - len(hdr))
            if not more:
                raise ConnectionError("channel closed")
            hdr += more
        n, n_fds = _HDR.unpack(hdr)
        fds = list(fds)
        while len(fds) < n_fds:
            mark, more, _, _ = socket.recv_fds(self.sock, 1, self.MAX_FDS)
            assert mark == b"+", mark
            fds += more
        buf = bytearray()
        while len(buf) < n:
            chunk = self.sock.recv(n - len(buf))
            if not chunk:
                raise ConnectionError("channel closed")
            buf += chunk
        assert len(fds) == n_fds, (len(fds), n_fds)
        return pickle.loads(bytes(buf)), list(fds)

    def close(self) -> None:
        self.sock.close()


def store_layout(store: KvStore) -> list[int]:
    out = np.zeros(8, dtype=np.int64)
    _check(N.lib().pl_store_layout(store._h, N.ptr(out)))
    return [int(x) for x in out]


def export_groups(store: KvStore, groups) -> tuple[dict, list[int]]:
    """(meta {group: (chunk_bytes, n_chunks, base)}, fds in group order)."""
    meta, fds = {}, []
    for g in sorted(groups):
        buf = (C.c_int * 4096)()
        n, cb = C.c_int(), C.c_int64()
        _check(N.lib().pl_store_export_group(store._h, g, buf, 4096, C.byref(n), C.byref(cb)))
        meta[g] = (cb.value, n.value, store.group_base(g))
        fds += list(buf[: n.value])
    return meta, fds


def export_table(store: KvStore) -> tuple[bytes, int, int]:
    h = (C.c_ubyte * 64)()
    mr, mc = C.c_int64(), C.c_int64()
    _check(N.lib().pl_store_export_table(store._h, h, C.byref(mr), C.byref(mc)))
    return bytes(h), mr.value, mc.value


def table_version(store: KvStore) -> tuple[int, int, int]:
    p, mr, mc = C.c_uint64(), C.c_int64(), C.c_int64()
    _check(N.lib().pl_store_table_version(store._h, C.byref(p), C.byref(mr), C.byref(mc)))
    return p.value, mr.value, mc.value


class RemoteStore:
    """This process's view of a peer process's store (pl_remote)."""

    def __init__(self, device: int, layout: list[int]) -> None:
        s, k, cell, fp, unit, groups = layout[:6]
        h = C.c_void_p()
        N.check(N.lib().pl_remote_create(device, s, k, cell, fp, unit, groups, C.byref(h)))
        self.h = h
        self.layout = layout

    def import_groups(self, meta: dict, fds: list[int]) -> None:
        i = 0
        for g, (cb, n, _base) in sorted(meta.items()):
            arr = (C.c_int * n)(*fds[i:i + n])
            N.check(N.lib().pl_remote_import_group(self.h, g, arr, n, cb))
            i += n
        for fd in fds:   # the driver holds its own reference after the import
            os.close(fd)

    def set_table(self, handle: bytes, max_reqs: int, max_chain: int) -> None:
        buf = (C.c_ubyte * 64).from_buffer_copy(handle)
        N.check(N.lib().pl_remote_set_table(self.h, buf, max_reqs, max_chain))

    def close(self, after_stream: int | None = None) -> None:
        """Tear the view down; with `after_stream`, on a background thread once the work
        enqueued on that stream (the last pushes through the view) has run."""
        if self.h is not None:
            if after_stream is not None:
                N.check(N.lib().pl_remote_destroy_after(self.h, C.c_void_p(after_stream)))
            else:
                N.lib().pl_remote_destroy(self.h)
            self.h = None


class PatchReceiver:
    """Destination half of a cross-process pair: maps the migrating groups, exports
    them, and serves patch rounds until the sender closes the pair."""

    def __init__(self, store: KvStore, groups, chan: Channel, mailbox: bool | None = None) -> None:
        self.store = store
        self.groups = sorted(groups)
        self.chan = chan
        # the round's control over a shared-memory mailbox (default) or socket messages
        # (PL_PATCH_SOCKET=1, the round-1 protocol kept for A/B timing)
        if mailbox is None:
            mailbox = os.environ.get("PL_PATCH_SOCKET") is None
        self.mb = Mailbox.create(store.device) if mailbox else None
        self.seq = 0
        self._groups_arr = N.as_i32(self.groups)
        self._versions = np.zeros(2, dtype=np.uint64)   # (table, pools) hashes, set below
        # ctypes arguments of the per-round calls, built once (numpy's .ctypes costs ~2 us)
        self._groups_p, self._versions_p = N.ptr(self._groups_arr), N.ptr(self._versions)
        self._flags, self._done = C.c_int(), C.c_int64()
        self._flags_ref, self._done_ref = C.byref(self._flags), C.byref(self._done)
        store.resident_groups |= set(self.groups)
        self._send_hello()
        self.rounds = 0
        self.items_reserved = 0
        self.table_reexports = 0   # block table reallocated mid-migration -> re-exported
        self.pool_reexports = 0

    def _pool_state(self):
        return tuple(self.store.group_base(g) for g in self.groups), self.store.info()["mapped_bytes"]

    def _send_hello(self) -> None:
        meta, fds = export_groups(self.store, self.groups)
        table = export_table(self.store)
        self._pools = self._pool_state()
        self._table = table_version(self.store)
        N.check(N.lib().pl_store_export_versions(self.store._h, N.ptr(self._groups_arr),
                                                 len(self.groups), N.ptr(self._versions)))
        self.chan.send(("hello", store_layout(self.store), meta, table,
                        self.mb.export() if self.mb is not None else None), fds)
        for fd in fds:
            os.close(fd)

    def _updates(self) -> tuple[dict, list[int]]:
        update, fds = {}, []
        if table_version(self.store) != self._table:
            update["table"] = export_table(self.store)
            self._table = table_version(self.store)
            self.table_reexports += 1
        if self._pool_state() != self._pools:
            update["pools"], fds = export_groups(self.store, self.groups)
            self._pools = self._pool_state()
            self.pool_reexports += 1
        return update, fds

    def serve(self) -> bool:
        """One round; False once the sender closed the pair."""
        if not self.serve_rows():
            return False
        self.serve_ack()
        return True

    def serve_rows(self) -> bool:
        """First half of a round: reserve the drained rows, publish table/pool updates."""
        if self.mb is not None:
            return self._serve_rows_mailbox()
        msg, _ = self.chan.recv()
        if msg[0] == "close":
            return False
        assert msg[0] == "rows", msg[0]
        reqs, groups, a, b = (np.ascontiguousarray(x) for x in msg[1])
        done = C.c_int64()
        rc = N.lib().pl_store_reserve_rows(self.store._h, len(reqs), N.ptr(reqs), N.ptr(groups),
                                           N.ptr(a), N.ptr(b), C.byref(done))
        err = None if rc == N.PL_OK else (rc, N.lib().pl_last_error().decode(errors="replace"))
        self.store.sync()   # the table is read by the sending process next
        update, fds = {}, []
        if table_version(self.store) != self._table:
            update["table"] = export_table(self.store)
            self._table = table_version(self.store)
            self.table_reexports += 1
        if self._pool_state() != self._pools:
            update["pools"], fds = export_groups(self.store, self.groups)
            self._pools = self._pool_state()
            self.pool_reexports += 1
        self.chan.send(("reserved", done.value, err, update), fds)
        for fd in fds:
            os.close(fd)
        self.rounds += 1
        self.items_reserved += done.value
        self._err = err
        return True

    def _serve_rows_mailbox(self) -> bool:
        # the whole receiver half in one native call (pl_pair_serve_rows): wait for the rows,
        # reserve them in place, record "reserved", reply -- unless the table or pools the
        # sender imported changed, in which case the re-export goes over the socket first
        self.seq += 1
        flags, done = self._flags, self._done
        rc = N.lib().pl_pair_serve_rows(self.store._h, self.mb.h, self._groups_p,
                                        len(self.groups), self.seq, 300_000,
                                        self._versions_p, self._flags_ref, self._done_ref)
        if flags.value & 1:
            return False
        err = None if rc == N.PL_OK else (rc, N.lib().pl_last_error().decode(errors="replace"))
        if err is not None and not flags.value & 8:   # the call failed (not the reservation)
            raise N.NativeError(rc, err[1])
        if flags.value & 6:   # rare (a reallocated table, re-mapped pools): over the socket
            update, fds = {}, []
            if flags.value & 2:
                update["table"] = export_table(self.store)
                self._table = table_version(self.store)
                self.table_reexports += 1
            if flags.value & 4:
                update["pools"], fds = export_groups(self.store, self.groups)
                self._pools = self._pool_state()
                self.pool_reexports += 1
            self.chan.send(("update", update), fds)
            for fd in fds:
                os.close(fd)
            N.check(N.lib().pl_store_export_versions(self.store._h, N.ptr(self._groups_arr),
                                                     len(self.groups), N.ptr(self._versions)))
            self.mb.post(W_REPLY, self.seq)
        self.rounds += 1
        self.items_reserved += done.value
        self._err = err
        return True

    def serve_ack(self) -> None:
        """Second half: the sender's cells are in this store once "applied" arrives
        (mailbox: this store's stream waits on the device for the sender's push)."""
        if self.mb is not None:
            N.check(N.lib().pl_pair_serve_ack(self.store._h, self.mb.h, self.seq, 300_000))
        else:
            ack, _ = self.chan.recv()
            assert ack[0] == "applied", ack[0]
        if self._err is not None:
            from .kvstore import _ERRORS
            err, self._err = self._err, None
            raise _ERRORS.get(err[0], N.NativeError)(err[1])


_RETIRED: list = []   # closed pairs' patch engines, inactive, destroyed by reap_patches()


def reap_patches() -> int:
    """Destroy the patch engines of closed pairs (synchronises their streams): at a point
    where a host wait is harmless -- the next reconfiguration's start, or teardown."""
    n = len(_RETIRED)
    while _RETIRED:
        _RETIRED.pop().close()
    return n


class PatchSender:
    """Source half of a cross-process pair: the native patch engine over the local store
    plus the remote view of the receiver's pools and table."""

    def __init__(self, store: KvStore, groups, layers_per_group: int, chan: Channel,
                 rank_fn) -> None:
        self.store = store
        self.chan = chan
        self.rank_fn = rank_fn            # () -> int32 rank of every request handle
        self.patch = NativePatch(store, groups, layers_per_group)
        msg, fds = chan.recv()
        assert msg[0] == "hello", msg[0]
        _, layout, meta, (th, mr, mc), mb_blob = msg
        self.remote = RemoteStore(store.device, layout)
        self.remote.import_groups(meta, fds)
        self.remote.set_table(th, mr, mc)
        self.mb = Mailbox.open(store.device, mb_blob) if mb_blob is not None else None
        self.seq = 0
        # ctypes arguments of the per-round calls, built once
        self._rank, self._rank_args = None, (None, 0)
        a = (C.c_int64(), C.c_int64(), C.c_int64())
        self._args = a + tuple(C.byref(x) for x in a)
        self._fin = (C.c_int(), C.c_int(), C.c_int64())
        self._fin_refs = tuple(C.byref(x) for x in self._fin)
        self.keys = self.cells = 0

    def seed(self) -> int:
        """MigrationStream.start (migrator.py:170-183): every live cell becomes dirty."""
        return self.patch.seed()

    def round(self) -> tuple[int, int]:
        """Drain + push one patch; returns (keys, cells) like MigrationStream._drain."""
        self.begin()
        return self.finish()

    def begin(self) -> None:
        """Drain (host snapshot + K3) and send the rows to the receiver."""
        rank = self.rank_fn()
        if self.mb is not None:
            # drain + rows into the shared region + post, in one native call
            if rank is not self._rank:
                self._rank, self._rank_args = rank, (N.ptr(rank), len(rank))
            self.seq += 1
            a = self._args
            N.check(N.lib().pl_pair_send_rows(self.patch.h, self.mb.h, *self._rank_args,
                                              self.seq, a[3], a[4], a[5]))
            self._pending = (a[0].value, a[1].value)
            return
        keys, cells, n = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lib().pl_patch_drain_rows(self.patch.h, N.ptr(rank), len(rank), C.byref(keys),
                                            C.byref(cells), C.byref(n)))
        m = n.value
        self._pending = (keys.value, cells.value)
        rows = (np.empty(m, np.int32), np.empty(m, np.int32), np.empty(m, np.int64),
                np.empty(m, np.int64))
        N.check(N.lib().pl_patch_rows(self.patch.h, *(N.ptr(x) for x in rows), m))
        self.chan.send(("rows", rows))

    def finish(self) -> tuple[int, int]:
        """Receive the reservation, push the cells into the remote pools, acknowledge."""
        if self.mb is not None:
            # wait for the reply, push into the remote pools, record + post "applied": one
            # native call, two when the receiver re-exported its table or pools
            need, rc, done = self._fin
            N.check(N.lib().pl_pair_finish(self.patch.h, self.remote.h, self.mb.h, self.seq,
                                           300_000, 0, *self._fin_refs))
            if need.value:
                (tag, update), fds = self.chan.recv()
                assert tag == "update", tag
                if "pools" in update:
                    self.remote.import_groups(update["pools"], fds)
                if "table" in update:
                    self.remote.set_table(*update["table"])
                N.check(N.lib().pl_pair_finish(self.patch.h, self.remote.h, self.mb.h, self.seq,
                                               300_000, 1, *self._fin_refs))
            err = None
            if rc.value != N.PL_OK:
                raw = bytes(np.ctypeslib.as_array((C.c_ubyte * 256).from_address(self.mb.base + 8 * W_MSG)))
                err = (rc.value, raw.split(b"\0", 1)[0].decode(errors="replace"))
        else:
            msg, fds = self.chan.recv()
            assert msg[0] == "reserved", msg[0]
            _, done, err, update = msg
            if "pools" in update:
                self.remote.import_groups(update["pools"], fds)
            if "table" in update:
                self.remote.set_table(*update["table"])
            N.check(N.lib().pl_patch_push_remote(self.patch.h, self.remote.h, done))
            self.store.sync()   # the cells are in the receiver's HBM before it is told so
            self.chan.send(("applied",))
        if err is not None:
            from .kvstore import _ERRORS
            raise _ERRORS.get(err[0], N.NativeError)(err[1])
        keys, cells = self._pending
        self.keys += keys
        self.cells += cells
        return keys, cells

    def dirty_keys(self) -> int:
        return self.patch.dirty_keys()

    def close(self) -> None:
        t = [time.perf_counter()]
        # the pushes into the remote pools were enqueued on the patch's stream: the view is
        # unmapped once they have run (background thread, no host wait here)
        push_stream = self.patch.stream_ptr()
        if self.mb is not None:
            self.mb.words[W_CLOSE] = 1
            self.seq += 1
            self.mb.post(W_ROWS, self.seq)
            t.append(time.perf_counter())
            self.mb.close()
        else:
            self.chan.send(("close",))
            t.append(time.perf_counter())
        t.append(time.perf_counter())
        self.remote.close(after_stream=push_stream)
        t.append(time.perf_counter())
        # the engine stops marking now; its device buffers are freed later (reap_patches:
        # destroying it here would synchronise its streams inside the decode loop)
        N.check(N.lib().pl_patch_set_active(self.patch.h, 0))
        _RETIRED.append(self.patch)
        t.append(time.perf_counter())
        self.close_phases_ms = {k: round((t[i + 1] - t[i]) * 1e3, 3) for i, k in
                                enumerate(("signal", "mailbox", "remote", "patch"))}


class ActRing:
    """A K7 activation ring (pl_act_ring, csrc/act.cu): device slots owned by the
    receiving stage, written by the sending stage, handed over with interprocess events
    and a shared-memory mailbox -- device to device, no host staging, no stream sync."""

    def __init__(self, h, device: int) -> None:
        self.h = h
        self.device = device

    @classmethod
    def create(cls, device: int, slot_bytes: int, n_slots: int = 4) -> "ActRing":
        h = C.c_void_p()
        N.check(N.lib().pl_act_ring_create(device, slot_bytes, n_slots, C.byref(h)))
        return cls(h, device)

    @classmethod
    def open(cls, device: int, blob: bytes) -> "ActRing":
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        h = C.c_void_p()
        N.check(N.lib().pl_act_ring_open(device, buf, len(blob), C.byref(h)))
        return cls(h, device)

    def export(self) -> bytes:
        n = C.c_int64()
        N.check(N.lib().pl_act_ring_export(self.h, None, 0, C.byref(n)))
        buf = (C.c_ubyte * n.value)()
        N.check(N.lib().pl_act_ring_export(self.h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def send(self, t, stream_ptr: int) -> None:
        N.check(N.lib().pl_act_send(self.h, C.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                                    C.c_void_p(stream_ptr)))

    def recv(self, t, stream_ptr: int) -> None:
        N.check(N.lib().pl_act_recv(self.h, C.c_void_p(t.data_ptr()), t.numel() * t.element_size(),
                                    C.c_void_p(stream_ptr)))

    def close(self) -> None:
        if self.h is not None:
            N.lib().pl_act_ring_destroy(self.h)
            self.h = None


class Mailbox:
    """pl_mailbox (csrc/act.cu): POSIX shared memory between the two processes of a pair
    plus interprocess CUDA events.  Words 0..63 are control words; the rest is a row area."""

    ROWS_OFF = 512

    def __init__(self, h, device: int) -> None:
        self.h = h
        self.device = device
        base, n = C.c_void_p(), C.c_int64()
        N.check(N.lib().pl_mailbox_base(h, C.byref(base), C.byref(n)))
        self.base, self.bytes = base.value, n.value
        self.cap = (self.bytes - self.ROWS_OFF) // 24
        off = self.base + self.ROWS_OFF
        self.reqs = np.ctypeslib.as_array((C.c_int32 * self.cap).from_address(off))
        self.groups = np.ctypeslib.as_array((C.c_int32 * self.cap).from_address(off + 4 * self.cap))
        self.a = np.ctypeslib.as_array((C.c_int64 * self.cap).from_address(off + 8 * self.cap))
        self.b = np.ctypeslib.as_array((C.c_int64 * self.cap).from_address(off + 16 * self.cap))
        self.words = np.ctypeslib.as_array((C.c_uint64 * 64).from_address(self.base))

    @classmethod
    def create(cls, device: int, rows: int = 1 << 18, n_events: int = 2) -> "Mailbox":
        h = C.c_void_p()
        N.check(N.lib().pl_mailbox_create(device, cls.ROWS_OFF + 24 * rows, n_events, C.byref(h)))
        return cls(h, device)

    @classmethod
    def open(cls, device: int, blob: bytes) -> "Mailbox":
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        h = C.c_void_p()
        N.check(N.lib().pl_mailbox_open(device, buf, len(blob), C.byref(h)))
        return cls(h, device)

    def export(self) -> bytes:
        n = C.c_int64()
        N.check(N.lib().pl_mailbox_export(self.h, None, 0, C.byref(n)))
        buf = (C.c_ubyte * n.value)()
        N.check(N.lib().pl_mailbox_export(self.h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def post(self, word: int, value: int) -> None:
        N.check(N.lib().pl_mailbox_post(self.h, word, value))

    def wait(self, word: int, at_least: int, timeout_ms: int = 300_000) -> int:
        out = C.c_uint64()
        N.check(N.lib().pl_mailbox_wait(self.h, word, at_least, timeout_ms, C.byref(out)))
        return out.value

    def record(self, event: int, stream_ptr: int) -> None:
        N.check(N.lib().pl_mailbox_record(self.h, event, C.c_void_p(stream_ptr)))

    def stream_wait(self, event: int, stream_ptr: int) -> None:
        N.check(N.lib().pl_mailbox_stream_wait(self.h, event, C.c_void_p(stream_ptr)))

    def close(self) -> None:
        if self.h is not None:
            N.lib().pl_mailbox_destroy(self.h)
            self.h = None


# control words of a patch pair's mailbox
W_ROWS, W_REPLY, W_APPLIED, W_NROWS, W_DONE, W_ERR, W_UPDATE, W_CLOSE = range(8)
W_MSG = 8            # words 8..39: error message bytes (256 B)
EV_APPLIED = 0       # interprocess event: the sender's push of the round (sender records)
EV_RESERVED = 1      # interprocess event: the receiver's table deltas of the round


class StageLink:
    """Stage-to-stage activations (K7, engine.py:353-375, fabric.py:129-136).

    mode "ring" (default): one ActRing per directed stage pair, created lazily by the
    receiver and handed to the sender over a local Channel -- device-to-device copies
    ordered on the stages' streams (NVLink between GPUs, HBM when they share one).
    mode "nccl": isend/irecv on the NCCL group (the stream waits, not the host).
    mode "gloo": blocking send/recv staged through host memory (CPU tests only)."""

    def __init__(self, group=None, mode: str | None = None, prefix: str = "pl",
                 device: int = 0, slot_bytes: int = 8 << 20) -> None:
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.backend = dist.get_backend(group)
        import torch

        # the device ring needs CUDA; CPU-only processes (gloo tests) stage through host memory
        self.mode = mode or os.environ.get("PL_ACT_MODE") or (
            "ring" if torch.cuda.is_available() else self.backend)
        self.rank = dist.get_rank(group)
        self.prefix = prefix
        self.device = device
        self.slot_bytes = slot_bytes
        self.rings: dict = {}    # (src, dst) -> ActRing
        self._keep = []          # tensors an in-flight NCCL isend still reads
        self.sent_bytes = 0

    def _stream(self) -> int:
        import torch
        return torch.cuda.current_stream(self.device).cuda_stream

    def _ring(self, src: int, dst: int) -> ActRing:
        key = (src, dst)
        r = self.rings.get(key)
        if r is None:
            name = f"{self.prefix}-act-{src}-{dst}"
            if dst == self.rank:   # the receiver owns the ring
                chan = Channel(name, server=True)
                r = ActRing.create(self.device, self.slot_bytes)
                chan.send(("ring", r.export()))
            else:
                chan = Channel(name, server=False)
                msg, _ = chan.recv()
                assert msg[0] == "ring", msg[0]
                r = ActRing.open(self.device, msg[1])
            chan.close()
            self.rings[key] = r
        return r

    def send(self, t, dst: int) -> None:
        t = t.contiguous()
        self.sent_bytes += t.numel() * t.element_size()
        if self.mode == "ring":
            self._ring(self.rank, dst).send(t, self._stream())
            self._keep = [t]          # the copy on the stream reads it
        elif self.backend == "nccl":
            self._keep = [t]
            self.dist.isend(t, dst, group=self.group)
        else:
            self.dist.send(t.detach().to("cpu"), dst, group=self.group)

    def recv(self, shape, dtype, src: int, device):
        import torch

        if self.mode == "ring":
            t = torch.empty(shape, dtype=dtype, device=device)
            self._ring(src, self.rank).recv(t, self._stream())
            return t
        if self.backend == "nccl":
            t = torch.empty(shape, dtype=dtype, device=device)
            self.dist.irecv(t, src, group=self.group).wait()   # the stream waits, not the host
            return t
        t = torch.empty(shape, dtype=dtype)
        self.dist.recv(t, src, group=self.group)
        return t.to(device)

    @property
    def host_staged(self) -> bool:
        return self.mode != "ring" and self.backend != "nccl"

    def close(self) -> None:
        for r in self.rings.values():
            r.close()
        self.rings.clear()


class RingPair:
    """Bench topology for N > 1 ranks (one per GPU): rank r's migrating groups stream to
    rank r+1, so every GPU sends one pair and receives one pair at the same time (N
    concurrent distinct-source pairs over NVSwitch).  The source is the
    PatchRig's stage store; the receiving store holds the previous rank's groups."""

    def __init__(self, rig, rank: int, world: int, tag: str) -> None:
        from .kvstore import KvStore

        wl = rig.wl
        nxt, prv = (rank + 1) % world, (rank - 1) % world
        cap = wl.batch * (wl.blocks_per_req + 2) + 64
        self.dst = KvStore(100 + rank, wl.k, wl.s, cap, (), num_groups=wl.model_groups,
                           cell_bytes=wl.cell_bytes, device=rig.device, registry=rig.registry)
        lis = Channel.listen(f"{tag}-{prv}-{rank}")
        out = Channel.connect(f"{tag}-{rank}-{nxt}")
        inn = lis.accept()
        self.rx = PatchReceiver(self.dst, wl.mig_groups, inn)          # sends hello
        self.tx = PatchSender(rig.src, wl.mig_groups, wl.k, out, rig.registry.rank)
        self.payload_bytes = wl.payload_bytes

    def use_stream(self, stream_ptr: int) -> None:
        N.check(N.lib().pl_store_set_stream(self.dst._h, C.c_void_p(stream_ptr)))

    def bulk_round(self) -> tuple[int, int]:
        """One ring step: every live cell of the migrating groups, both directions."""
        self.tx.seed()
        self.tx.begin()
        self.rx.serve_rows()
        keys, cells = self.tx.finish()
        self.rx.serve_ack()
        return keys, cells

    def close(self) -> None:
        N.check(N.lib().pl_patch_set_active(self.tx.patch.h, 0))
        self.tx.close()
        assert not self.rx.serve()
        reap_patches()   # teardown: the closed pair's engine can synchronise now
