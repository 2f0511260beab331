"""The N>1 control plane of the cross-process patch path on CPU (gloo ranks, no GPU):
DistStagedLlama.start_reconfig / pump / post_commit open one dist.Channel per migrating
(src, dst) pair in ONE global pair order on every rank, the receiver sends its exported
pool chunks as file descriptors (SCM_RIGHTS, more than one message's worth here), and
every round walks the pairs in that same order.  Eight ranks run the BASELINE configs[3]
re-split (even -> uneven, six pairs, four ranks both send and receive) and a world-size-2
pair; stand-in payloads (memfds, interval rows) replace the device parts, so what is
tested is the host protocol: no rank waits on a peer that waits on it, descriptors and
rows arrive intact, the close handshake ends every pair."""

import os
import socket

import pytest
import torch.multiprocessing as mp

import dist_workers as W


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _memfd(tag: str) -> int:
    fd = os.memfd_create(tag)
    os.write(fd, tag.encode())
    return fd


def _rank(rank, world, port, prefix, src_conf, dst_conf, n_fds, rounds, out):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2604_12171_b200.dist import Channel
        from paper_2604_12171_b200.llama import layer_moves

        gpu = rank + 1
        owner = {l: g for g, ls in src_conf.items() for l in ls}
        moves = layer_moves(owner, dst_conf)
        pairs = sorted(moves)
        chans, got = {}, []
        # setup in the global pair order (start_reconfig): the receiver listens, accepts and
        # sends its "hello" with the pool fds; the sender connects and reads it
        for (src, dst) in pairs:
            name = f"{prefix}-{src}-{dst}"
            if dst == gpu:
                ch = Channel(name, server=True)
                fds = [_memfd(f"{dst}:{l}:{i}") for l in moves[(src, dst)] for i in range(n_fds)]
                ch.send(("hello", moves[(src, dst)]), fds)
                for fd in fds:
                    os.close(fd)
                chans[(src, dst)] = ch
            elif src == gpu:
                ch = Channel(name, server=False)
                (tag, layers), fds = ch.recv()
                assert tag == "hello" and layers == moves[(src, dst)]
                want = [f"{dst}:{l}:{i}" for l in layers for i in range(n_fds)]
                seen = []
                for fd in fds:
                    os.lseek(fd, 0, os.SEEK_SET)
                    seen.append(os.read(fd, 64).decode())
                    os.close(fd)
                assert seen == want, (seen[:3], want[:3])
                got.append(("fds", (src, dst), len(fds)))
                chans[(src, dst)] = ch
        # rounds (pump): sender -> rows, receiver -> reply, sender -> applied, pair by pair
        for r in range(rounds):
            for (src, dst) in pairs:
                if src == gpu:
                    ch = chans[(src, dst)]
                    rows = [(req, (src * 7 + req) % 3, r * 16, r * 16 + 16) for req in range(8)]
                    ch.send(("rows", rows))
                    (tag, n), _ = ch.recv()
                    assert tag == "reserved" and n == len(rows)
                    ch.send(("applied", r))
                elif dst == gpu:
                    ch = chans[(src, dst)]
                    (tag, rows), _ = ch.recv()
                    assert tag == "rows" and rows[0] == (0, (src * 7) % 3, r * 16, r * 16 + 16)
                    ch.send(("reserved", len(rows)))
                    (tag, rr), _ = ch.recv()
                    assert tag == "applied" and rr == r
                    got.append(("round", (src, dst), r))
        # post-commit close in the same order
        for (src, dst) in pairs:
            if src == gpu:
                chans[(src, dst)].send(("close",))
                chans[(src, dst)].close()
            elif dst == gpu:
                (tag,), _ = chans[(src, dst)].recv()
                assert tag == "close"
                chans[(src, dst)].close()
        dist.barrier()
        out.put((rank, "ok", got))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        out.put((rank, "error", traceback.format_exc()))


def _run(world, src_conf, dst_conf, n_fds, rounds):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    prefix = f"cpu-pairs-{os.getpid()}-{port}"
    procs = [ctx.Process(target=_rank, args=(r, world, port, prefix, src_conf, dst_conf, n_fds,
                                             rounds, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=180)
        assert r[1] == "ok", r[2]
        res[r[0]] = r[2]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_eight_rank_uneven_resplit_pairs_in_global_order():
    from paper_2604_12171_b200.llama import layer_moves

    owner = {l: g for g, ls in W.CONF_EVEN8.items() for l in ls}
    moves = layer_moves(owner, W.CONF_UNEVEN8)
    assert len(moves) == 6   # four ranks both send and receive
    res = _run(8, W.CONF_EVEN8, W.CONF_UNEVEN8, n_fds=130, rounds=3)
    rounds = sorted(x for g in res.values() for x in g if x[0] == "round")
    assert rounds == sorted(("round", p, r) for p in moves for r in range(3))
    fds = sorted(x for g in res.values() for x in g if x[0] == "fds")
    assert fds == sorted(("fds", p, 130 * len(ls)) for p, ls in moves.items())


@pytest.mark.parametrize("n_fds", [1, 300])
def test_world_size_two_pair(n_fds):
    # layer 3 moves from GPU 2 (rank 1, sender) to GPU 1 (rank 0, receiver)
    res = _run(2, W.CONF_A, {1: [1, 2, 3], 2: [4]}, n_fds=n_fds, rounds=4)
    assert res[0] == [("round", (2, 1), r) for r in range(4)]
    assert res[1] == [("fds", (2, 1), n_fds)]
