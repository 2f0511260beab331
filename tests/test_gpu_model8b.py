"""BASELINE configs[1] with real stage compute (paper_2604_12171_b200/model8b.py): a
Llama-3-8B-shaped decoder (bf16 weights, tensor-core GEMMs, K1/K2 over the stage stores)
decodes greedily while a live PP 2 -> 4 reconfiguration moves layers 9-16 and 25-32 on
side streams; the switch is taken at the first per-step poll with lag < tau (the
reference's safe-switch test, migrator.py:341-348).  The tokens must equal the static
run's, and the moved groups' KV on the destinations must equal the source's bytes."""

import pytest

pytestmark = pytest.mark.gpu


def test_live_pp2_to_pp4_tokens_equal_static_small_batch():
    from paper_2604_12171_b200.model8b import PP4, run_live, summarize

    kw = dict(batch=16, ctx=256, steps=14, reconfig_at=4)
    static = run_live(live=False, **kw)
    live = run_live(live=True, **kw)
    s = summarize(live, static)
    assert s["tokens_equal_static"], (live["tokens"], static["tokens"])
    assert s["switch_step"] is not None and s["switch_step"] > 4
    assert s["commit"]["lag_at_poll"] < 50
    assert live["config_end"] == {g: PP4[g] for g in sorted(PP4)}
    # the bulk round after step 4: 16 requests x (256 + 5) positions x 2 pairs x 2 groups x k
    assert s["steps_per_phase"]["after"] > 0 and s["bulk"]["cells"] == 16 * 261 * 4 * 4
    print(s)


def test_live_even8_to_uneven8_tokens_equal_static_small_batch():
    """configs[3] at the 8B shape: 8 stage stores, even 4-layer split -> 2/4/4/6/6/4/4/2
    at k = 2, six pairs (stages 2, 3, 6, 7 send and receive) patch concurrently; the switch
    is the first poll with lag < tau, and the tokens equal the static run's."""
    from paper_2604_12171_b200.llama import layer_moves
    from paper_2604_12171_b200.model8b import EVEN8, UNEVEN8, run_live, summarize

    kw = dict(batch=8, ctx=128, steps=12, reconfig_at=3, src=EVEN8, dst=UNEVEN8, k=2)
    static = run_live(live=False, **kw)
    live = run_live(live=True, **kw)
    s = summarize(live, static)
    assert s["tokens_equal_static"], (live["tokens"], static["tokens"])
    assert s["switch_step"] is not None and s["switch_step"] > 3
    assert s["commit"]["lag_at_poll"] < 50
    assert live["config_end"] == {g: UNEVEN8[g] for g in sorted(UNEVEN8)}
    moves = layer_moves({l: g for g, ls in EVEN8.items() for l in ls}, UNEVEN8)
    assert len(moves) == 6
    # bulk: every moved layer group of the 8 requests at 128 + 4 positions, k = 2 cells
    assert s["bulk"]["cells"] == 8 * 132 * 2 * len(moves)
