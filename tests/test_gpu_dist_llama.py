"""The tiny Llama with one process per pipeline stage (3 ranks on one GPU): hidden states
cross stages device to device through the K7 activation rings (csrc/act.cu: IPC
buffers + interprocess events, no host staging), and a live PP 2 -> 3 reconfiguration
moves layer 2 (rank 0 -> 1) and layer 4 (rank 1 -> 2) with the cross-process push.  The
stage compute runs in exact mode, so the greedy tokens must equal the CPU oracle's
(oracle/llama_exact.c) and the single-process run, bit for bit."""

import multiprocessing as mp
import os
import socket

import pytest

import dist_workers as W

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_dist(live, target=None, world=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    prefix = f"dl-{os.getpid()}-{port}"
    procs = [ctx.Process(target=target or W.stage, args=(r, world, port, prefix, q, live))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=300)
        assert r[1] != "error", r[2]
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_process_per_stage_live_reconfig_matches_oracle():
    from oracle.llama import ExactOracleLlama
    from paper_2604_12171_b200.llama import LlamaConfig, StagedLlama, generate, init_weights

    cfg = LlamaConfig()
    want = ExactOracleLlama(cfg, init_weights(cfg, 0)).generate(W.PROMPTS, W.JOINS, W.N_GEN)
    m = StagedLlama(cfg, init_weights(cfg, 0), W.CONF_A, exact=True)
    assert generate(m, W.PROMPTS, W.JOINS, W.N_GEN) == want
    static = _run_dist(False)
    live = _run_dist(True)
    conv = _run_dist("converged")   # switch decided by the dirty-set threshold (tau = 50)
    for r in range(3):
        assert static[r][0] == want
        assert live[r][0] == want
        assert conv[r][0] == want
        assert conv[r][1] == live[r][1]
        # activations moved device to device (K7 rings), none through host memory
        assert live[r][2]["mode"] == "ring" and not live[r][2]["host_staged"]
    assert sum(live[r][2]["sent_bytes"] for r in range(3)) > 0
    # after the switch: rank 0 keeps layer 1, rank 1 layers 2-3, rank 2 layer 4
    assert live[0][1] == [0] and live[1][1] == [1, 2] and live[2][1] == [3]


def test_eight_stage_uneven_resplit_matches_oracle():
    """BASELINE configs[3] shape: 8 stage processes, a 16-layer model split evenly, re-split
    live into an uneven split: 6 pairs move a layer each, concurrently; ranks 2, 3, 6 and
    7 send one layer while receiving another (the global pair order keeps this
    deadlock-free)."""
    from oracle.llama import ExactOracleLlama
    from paper_2604_12171_b200.llama import LlamaConfig, init_weights

    cfg = LlamaConfig(n_layers=16)
    want = ExactOracleLlama(cfg, init_weights(cfg, 1)).generate(W.PROMPTS, W.JOINS, W.N_GEN)
    live = _run_dist(True, target=W.stage8, world=8)
    for r in range(8):
        assert live[r][0] == want, r
        assert live[r][3]["mode"] == "ring" and not live[r][3]["host_staged"]
    for g, layers in W.CONF_UNEVEN8.items():
        assert live[g - 1][1] == [l - 1 for l in layers]
