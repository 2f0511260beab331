"""The N>1 plumbing of bench.py on CPU: two gloo ranks, barrier, max-over-ranks timing,
and the rule that only rank 0 reports (the reference arm's other ranks exit quietly)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), LOCAL_RANK=str(rank))
    import bench

    r, w = bench.dist_init(world)
    bench.barrier(w)
    got = bench.allmax(float(10 * (r + 1)), w)
    out.put((r, w, got))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_two_rank_allmax_and_barrier():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, 2, 20.0), (1, 2, 20.0)]


def _ref_worker(rank, world, port, out):
    import contextlib
    import io
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import bench
    from paper_2604_12171_b200.perf import Workload

    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        if rank == 1:  # non-zero ranks of the reference arm do no work
            class A:
                steps, warmup = 1, 1
            bench.run_reference(A, Workload(batch=4, ctx=64), rank, world)
    out.put((rank, buf.getvalue()))


def test_reference_arm_silent_on_nonzero_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ref_worker, args=(1, 2, _free_port(), q))
    p.start()
    rank, text = q.get(timeout=120)
    p.join(timeout=60)
    assert p.exitcode == 0 and rank == 1 and text == ""
