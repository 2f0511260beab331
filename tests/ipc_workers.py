"""Worker processes of the cross-process patch tests (tests/test_gpu_ipc.py): both run
on cuda:0, in separate processes, exactly like two stage processes on two GPUs."""

import random

K, S, CELL, CAP = 2, 16, 256, 2048


def n_req(seed):
    # seeds >= 100: more requests than the receiver's initial block-table rows (64), so
    # its table is reallocated mid-migration and re-exported to the sender
    return 90 if seed >= 100 else 12


def names(seed):
    return [f"r{i:04d}" for i in range(n_req(seed))]


def _registry(seed):
    from paper_2604_12171_b200 import kvstore
    reg = kvstore.RequestRegistry()
    for n in names(seed):      # both processes assign the same handles
        reg.handle(n)
    return reg


def ops(seed):
    """(initial fill, per-round decode/prefill writes) of the source stage"""
    rng = random.Random(seed)
    nm = names(seed)
    fill = [(n, g, 5 + rng.randrange(60)) for n in nm[: len(nm) // 2] for g in range(4)]
    rounds = []
    for _ in range(4):
        w = []
        for n in rng.sample(nm, min(len(nm) - 1, 40)):   # includes requests that join later
            for g in rng.sample(range(4), 2):
                w.append((n, g, 1 + rng.randrange(20)))
        rounds.append(w)
    return fill, rounds


def src_store(reg):
    from paper_2604_12171_b200 import kvstore
    return kvstore.KvStore(1, K, S, CAP, (0, 1, 2, 3), num_groups=4, cell_bytes=CELL, registry=reg)


def dst_store(reg, cap=CAP):
    from paper_2604_12171_b200 import kvstore
    return kvstore.KvStore(2, K, S, cap, (), num_groups=4, cell_bytes=CELL, registry=reg)


# a destination too small for the bulk round: the receiver's reservation fails mid-round
CAP_SMALL = 5   # < one block per request of the fill: the round must overflow


def apply_writes(st, writes, mark):
    from paper_2604_12171_b200.events import stable_hash
    for n, g, cnt in writes:
        st.append_seeded(n, g, cnt, stable_hash(n, g), mark=mark)


def summary(st, groups=(2, 3)):
    snaps = {g: st.snapshot_group(g) for g in groups}
    cells = {}
    for g in groups:
        for rid, fps in snaps[g].items():
            for pos in {0, len(fps) // 2, len(fps) - 1}:
                for j in range(K):
                    cells[(rid, g, pos, j)] = st.read_cell(rid, g, pos, j)
    return snaps, cells, repr(st.state_digest())


def receiver(q, chan_name, seed):
    try:
        import torch
        torch.cuda.set_device(0)
        from paper_2604_12171_b200 import dist as D
        reg = _registry(seed)
        st = dst_store(reg)
        chan = D.Channel(chan_name, server=True)
        rx = D.PatchReceiver(st, [2, 3], chan)
        while rx.serve():
            pass
        q.put(("rx", summary(st), rx.rounds, rx.table_reexports))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(("rx-error", traceback.format_exc(), repr(e)))


def sender(q, chan_name, seed):
    try:
        import torch
        torch.cuda.set_device(0)
        from paper_2604_12171_b200 import dist as D
        reg = _registry(seed)
        st = src_store(reg)
        fill, rounds = ops(seed)
        apply_writes(st, fill, mark=False)
        chan = D.Channel(chan_name, server=False)
        tx = D.PatchSender(st, [2, 3], K, chan, reg.rank)
        tx.seed()
        log = [tx.round()]
        for w in rounds:
            apply_writes(st, w, mark=True)
            log.append(tx.round())
        tx.close()
        q.put(("tx", summary(st), log))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("tx-error", traceback.format_exc(), repr(e)))


def single_process(seed):
    """The same rounds with both stores in one process (local fused push)."""
    from paper_2604_12171_b200.perf import NativePatch
    reg = _registry(seed)
    src, dst = src_store(reg), dst_store(reg)
    dst.resident_groups |= {2, 3}
    fill, rounds = ops(seed)
    apply_writes(src, fill, mark=False)
    p = NativePatch(src, [2, 3], K)
    p.seed()
    log = [p.push(dst, reg.rank())]
    for w in rounds:
        apply_writes(src, w, mark=True)
        log.append(p.push(dst, reg.rank()))
    p.close()
    return summary(src), summary(dst), log


def receiver_overflow(q, chan_name, seed):
    """The receiver of a bulk round that overflows its pool: the reservation stops at the
    failing write (migrator.py:124-131), the round is still served, the error surfaces."""
    try:
        import torch
        torch.cuda.set_device(0)
        from paper_2604_12171_b200 import dist as D
        from paper_2604_12171_b200 import kvstore
        reg = _registry(seed)
        st = dst_store(reg, CAP_SMALL)
        chan = D.Channel(chan_name, server=True)
        rx = D.PatchReceiver(st, [2, 3], chan)
        errors = []
        while True:
            try:
                if not rx.serve():
                    break
            except kvstore.KvOverflow as e:
                errors.append(type(e).__name__)
        q.put(("rx", summary(st), rx.rounds, errors))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(("rx-error", traceback.format_exc(), repr(e)))


def sender_overflow(q, chan_name, seed):
    try:
        import torch
        torch.cuda.set_device(0)
        from paper_2604_12171_b200 import dist as D
        from paper_2604_12171_b200 import kvstore
        reg = _registry(seed)
        st = src_store(reg)
        fill, _ = ops(seed)
        apply_writes(st, fill, mark=False)
        chan = D.Channel(chan_name, server=False)
        tx = D.PatchSender(st, [2, 3], K, chan, reg.rank)
        tx.seed()
        errors = []
        try:
            tx.round()
        except kvstore.KvOverflow as e:
            errors.append(type(e).__name__)
        tx.close()
        q.put(("tx", errors))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("tx-error", traceback.format_exc(), repr(e)))


def single_process_overflow(seed):
    """The same overflowing bulk round with both stores in one process."""
    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200.perf import NativePatch
    reg = _registry(seed)
    src, dst = src_store(reg), dst_store(reg, CAP_SMALL)
    dst.resident_groups |= {2, 3}
    fill, _ = ops(seed)
    apply_writes(src, fill, mark=False)
    p = NativePatch(src, [2, 3], K)
    p.seed()
    code = None
    try:
        p.push(dst, reg.rank())
    except N.NativeError as e:
        code = e.code
    dst.sync()
    p.close()
    return summary(dst), code
