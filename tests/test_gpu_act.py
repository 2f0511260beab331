"""K7 activation rings and the pair mailbox (csrc/act.cu) in one process (the opened ring
aliases the owner's buffers; tests/test_gpu_dist_llama.py runs them across processes):
ordered hand-off of more activations than slots with the slot-reuse waits, device-side
ordering only (no stream sync between send and recv), and the mailbox's post / wait /
interprocess-event ordering."""

import pytest

pytestmark = pytest.mark.gpu


def test_ring_hands_off_in_order_across_slot_reuse():
    import torch

    from paper_2604_12171_b200.dist import ActRing

    owner = ActRing.create(0, 1 << 16, n_slots=3)
    sender = ActRing.open(0, owner.export())
    s_tx, s_rx = torch.cuda.Stream(), torch.cuda.Stream()
    sent, got = [], []
    for i in range(10):
        with torch.cuda.stream(s_tx):
            x = torch.full((64, 128), float(i), device="cuda") + torch.arange(128, device="cuda")
            torch.cuda._sleep(100_000)        # the copy is still queued when recv is called
        sent.append(x)
        sender.send(x, s_tx.cuda_stream)
        y = torch.empty(64, 128, device="cuda")
        owner.recv(y, s_rx.cuda_stream)
        got.append(y)
    torch.cuda.synchronize()
    for x, y in zip(sent, got):
        assert torch.equal(x, y)
    sender.close()
    owner.close()


def test_ring_rejects_oversized_activation():
    import torch

    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200.dist import ActRing

    owner = ActRing.create(0, 1024, n_slots=2)
    x = torch.zeros(1024, device="cuda")   # 4 KiB > 1 KiB slot
    with pytest.raises(N.NativeError):
        ActRing.open(0, owner.export()).send(x, torch.cuda.current_stream().cuda_stream)
    owner.close()


def test_mailbox_post_wait_and_event_ordering():
    import torch

    from paper_2604_12171_b200.dist import Mailbox

    own = Mailbox.create(0, rows=1024)
    peer = Mailbox.open(0, own.export())
    assert peer.cap == own.cap >= 1024
    peer.reqs[:4] = [7, 8, 9, 10]
    peer.post(0, 1)
    assert own.wait(0, 1) == 1 and list(own.reqs[:4]) == [7, 8, 9, 10]
    # an event recorded by one side orders the other side's stream on the device
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    buf = torch.zeros(1 << 20, device="cuda")
    with torch.cuda.stream(a):
        torch.cuda._sleep(200_000)
        buf.fill_(3.0)
    peer.record(0, a.cuda_stream)
    own.stream_wait(0, b.cuda_stream)
    with torch.cuda.stream(b):
        out = buf * 2
    torch.cuda.synchronize()
    assert float(out.min()) == 6.0
    peer.close()
    own.close()
