"""Cross-process KV patching on one GPU: the source and destination stages run in two
processes (as they would on two GPUs), the destination's pools are exported as VMM
fds + its block table as a CUDA IPC handle, and the fused push kernel writes the
destination's cells through the imported view.  The result must equal, bit for bit,
the single-process push of the same rounds (block ids, chains, fingerprints, KV bytes)
and the source's own copy of the migrated groups."""

import multiprocessing as mp
import os

import pytest

import ipc_workers as W
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,socket", [(0, False), (1, False), (100, False), (0, True),
                                         (100, True)])
def test_two_process_push_matches_single_process(seed, socket, monkeypatch):
    # the round's control over the shared-memory mailbox (default) or socket messages
    if socket:
        monkeypatch.setenv("PL_PATCH_SOCKET", "1")
    else:
        monkeypatch.delenv("PL_PATCH_SOCKET", raising=False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"ipc-test-{os.getpid()}-{seed}"
    procs = [ctx.Process(target=W.receiver, args=(q, name, seed)),
             ctx.Process(target=W.sender, args=(q, name, seed))]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=120)
        assert not r[0].endswith("error"), r[1]
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (tx_sum, tx_log), (rx_sum, rx_rounds, table_reexports) = res["tx"], res["rx"]
    assert rx_rounds == len(tx_log) == 5
    if W.n_req(seed) > 64:   # the receiver's block table grew mid-migration
        assert table_reexports >= 1
    src_sum, dst_sum, log = W.single_process(seed)
    assert [tuple(x) for x in tx_log] == [tuple(x) for x in log]   # keys, cells per round
    assert rx_sum == dst_sum                 # snapshots, sampled cells, full state digest
    assert rx_sum[0] == tx_sum[0]            # the destination holds the source's groups
    for (rid, g, pos, j), cell in rx_sum[1].items():
        fp = rx_sum[0][g][rid][pos]
        assert cell == oracle.expand_cell(fp, j, W.CELL)


@pytest.mark.parametrize("socket", [False, True])
def test_two_process_overflow_applies_the_same_prefix(socket, monkeypatch):
    """A bulk round the receiver cannot hold: across processes the receiver reserves up to
    the failing write, the sender pushes exactly that prefix, and both sides raise
    KvOverflow -- the destination ends identical to the single-process push of the same
    round (which applies the same prefix and returns the same error)."""
    if socket:
        monkeypatch.setenv("PL_PATCH_SOCKET", "1")
    else:
        monkeypatch.delenv("PL_PATCH_SOCKET", raising=False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"ipc-ovf-{os.getpid()}-{int(socket)}"
    procs = [ctx.Process(target=W.receiver_overflow, args=(q, name, 0)),
             ctx.Process(target=W.sender_overflow, args=(q, name, 0))]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=120)
        assert not r[0].endswith("error"), r[1]
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (tx_errors,), (rx_sum, rx_rounds, rx_errors) = res["tx"], res["rx"]
    assert rx_rounds == 1 and rx_errors == ["KvOverflow"] and tx_errors == ["KvOverflow"]
    dst_sum, code = W.single_process_overflow(0)
    assert code == -1                       # PL_E_KV_OVERFLOW
    assert rx_sum == dst_sum                # same prefix: snapshots, cells, state digest
    assert 0 < sum(len(v) for v in rx_sum[0][2].values())   # something was applied
