"""CPU checks of the process-per-GPU plumbing (dist.py, llama.py): the local control
channel with SCM_RIGHTS fd passing (the receiver's exported VMM chunks travel this way),
stage activations over a two-rank gloo group, and the pipeline-order / M_mig helpers."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _channel_server(name, n_fds, q):
    from paper_2604_12171_b200.dist import Channel
    pipes = [os.pipe() for _ in range(n_fds)]
    ch = Channel(name, server=True)
    ch.send(("hello", list(range(5))), [w for _, w in pipes])
    for _, w in pipes:
        os.close(w)
    # the peer writes one byte into every write end it received
    got = [os.read(r, 1) for r, _ in pipes]
    msg, _ = ch.recv()
    q.put((got, msg))


def _channel_client(name):
    from paper_2604_12171_b200.dist import Channel
    ch = Channel(name, server=False)
    msg, fds = ch.recv()
    assert msg == ("hello", [0, 1, 2, 3, 4])
    for i, fd in enumerate(fds):
        os.write(fd, bytes([i % 251]))
        os.close(fd)
    ch.send(("done", len(fds)))


@pytest.mark.parametrize("n_fds", [3, 300])   # 300 > one SCM_RIGHTS message
def test_channel_passes_objects_and_fds(n_fds):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"test-chan-{os.getpid()}-{n_fds}"
    s = ctx.Process(target=_channel_server, args=(name, n_fds, q))
    c = ctx.Process(target=_channel_client, args=(name,))
    s.start()
    c.start()
    got, msg = q.get(timeout=60)
    s.join(timeout=30)
    c.join(timeout=30)
    assert s.exitcode == 0 and c.exitcode == 0
    assert msg == ("done", n_fds)
    assert got == [bytes([i % 251]) for i in range(n_fds)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stage(rank, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2604_12171_b200.dist import StageLink
    link = StageLink()
    x = torch.arange(12, dtype=torch.float32).reshape(3, 4)
    if rank == 0:                    # stage 0 -> stage 1 -> stage 0 (the token loop)
        link.send(x * 2, 1)
        back = link.recv((3,), torch.int64, 1, "cpu")
        q.put((rank, back.tolist()))
    else:
        h = link.recv((3, 4), torch.float32, 0, "cpu")
        link.send(h.argmax(-1), 0)
        q.put((rank, h.sum().item()))
    dist.destroy_process_group()


def test_stage_link_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stage, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] == 2 * sum(range(12))
    assert res[0] == [3, 3, 3]


def test_pipeline_order_and_moves():
    from paper_2604_12171_b200.llama import layer_moves, pipeline_order

    owner = {1: 1, 2: 1, 3: 2, 4: 2}           # <1:[1,2], 2:[3,4], 3:{}>
    assert pipeline_order(owner) == [1, 2]
    moves = layer_moves(owner, {1: [1], 2: [2, 3], 3: [4]})
    assert moves == {(1, 2): [2], (2, 3): [4]}
    # pipeline reordering is legal: stage order follows the first layer
    assert pipeline_order({1: 2, 2: 2, 3: 1, 4: 1}) == [2, 1]
    with pytest.raises(ValueError):
        layer_moves(owner, {1: [1, 2], 2: [3]})
