"""The reference's acceptance criteria not covered elsewhere (pkg/tests/test_acceptance.py):
1 (block-budget oracle), 2 (config algebra), 5 (deadlock freedom), 7 (KV-resize
ablation), 8 (stacking trade-off), 9 (live switch beats every static config) and
10 (determinism).  Criteria 3, 4 and 6 are in test_gpu_kvstore.py / test_gpu_simulation.py.
1, 2 and 5 are host logic (CPU); 7-10 run whole scenarios on the GPU data plane."""

import random
import time
from fractions import Fraction
from math import ceil, floor

import pytest

import sim_scenarios as S

MIB = 1024 * 1024


def test_criterion_1_max_blocks_oracle():
    from paper_2604_12171_b200.cluster import GpuSpec, ModelSpec, max_blocks
    rng = random.Random(1001)
    t0 = time.time()
    for _ in range(1000):
        gran = rng.choice([1, 2, 4]) * MIB
        k = rng.choice([1, 2, 4])
        mem = gran * rng.randint(64, 65536)
        u = rng.choice([0.5, 0.75, 0.9, 0.95, 1.0])
        n = rng.randint(1, 64)
        w = rng.randint(0, mem // max(1, n))
        got = max_blocks(GpuSpec(1, mem, 1.0, 1.0, 1.0, gran), n, ModelSpec(n * k, w, 1, k), u)
        # exact rational budget: floor((M u - L W) / (L granularity / k)), None below zero
        num = Fraction(mem) * Fraction(u) - n * w
        assert got == (None if num < 0 else floor(num / (n * Fraction(gran, k))))
    assert time.time() - t0 < 1.0


def test_criterion_2_config_algebra_oracle():
    from paper_2604_12171_b200.cluster import PPConfig, diff_configs
    from test_reference_host_suites import _config
    rng = random.Random(2002)
    for _ in range(1000):
        n = rng.randint(2, 5)
        k = rng.choice([1, 2, 4])
        n_groups = rng.randint(n, 12)
        ids = list(range(1, n + 1))
        cur, tgt = _config(rng, ids, n_groups, k), _config(rng, ids, n_groups, k)
        c_int, m_add, m_del, m_mig = diff_configs(cur, tgt)
        a, b = cur.as_layer_sets(), tgt.as_layer_sets()
        for g in a:
            assert a[g] | m_add.get(g, set()) == c_int[g] and c_int[g] - m_del.get(g, set()) == b[g]
        moved = set()
        for (s, d), layers in m_mig.items():
            assert s != d and layers <= a[s] and layers <= m_add[d] and not moved & layers
            moved |= layers
        assert moved == (set().union(*m_add.values()) if m_add else set())
    assert diff_configs(S.C_A, S.C_B)[3] == {(1, 2): {2}, (2, 3): {4}}
    assert isinstance(S.C_A, PPConfig)


def test_criterion_5_deadlock():
    from paper_2604_12171_b200.fabric import detect_deadlock
    from test_reference_host_suites import fabric_, fig6, random_schedule
    sched, _, fab = fabric_(handshake=False)
    fig6(fab)
    sched.run()
    cycle = detect_deadlock(fab)
    assert cycle is not None and {g for g, _ in cycle} == {1, 2}
    t0 = time.time()
    for seed in range(10_000):
        f, ts = random_schedule(seed, True)
        assert detect_deadlock(f) is None and all(t.state == "done" for t in ts), seed
    assert time.time() - t0 < 120.0


@pytest.mark.gpu
def test_criterion_7_kv_resize_ablation():
    from paper_2604_12171_b200 import FeatureFlags, run_scenario
    on = run_scenario(S.hetero_scenario(rate=7.0), seed=7).metrics
    off = run_scenario(S.hetero_scenario(rate=7.0, flags=FeatureFlags(kv_resize=False)), seed=7).metrics
    assert on.overflow_events == 0 < off.overflow_events
    assert off.ttft_mean > on.ttft_mean


@pytest.mark.gpu
def test_criterion_8_stacking_tradeoff():
    from paper_2604_12171_b200 import enumerate_pp_configs, run_scenario
    util = {}
    for k in (1, 2, 4, 8):
        scen = S.stacking_scenario(k)
        u = run_scenario(scen, seed=11).metrics.effective_kv_utilization
        tokens = 512 + 16
        s = scen.model.tokens_per_block(scen.cluster[0])
        assert u == pytest.approx(tokens / (ceil(tokens / s) * s), abs=1e-12)
        assert u >= tokens / (tokens + s - 1)
        util[k] = u
    assert util[1] <= util[2] <= util[4] <= util[8]
    assert len(enumerate_pp_configs(16, 8, [1, 2])) < len(enumerate_pp_configs(16, 1, [1, 2]))


@pytest.mark.gpu
def test_criterion_9_live_switch_benefit():
    from paper_2604_12171_b200 import enumerate_pp_configs, run_scenario, score
    rows = [run_scenario(S.hetero_scenario(triggers=False, init=cfg), seed=7).metrics
            for cfg in enumerate_pp_configs(16, 2, [1, 2])]
    live = run_scenario(S.hetero_scenario(), seed=7)
    assert live.statuses and live.statuses[0].outcome == "success"
    scores = score(rows + [live.metrics])
    assert scores[-1] > max(scores[:-1])


@pytest.mark.gpu
def test_criterion_10_determinism():
    from paper_2604_12171_b200 import run_scenario
    a, b = (run_scenario(S.hetero_scenario(rate=7.0, n=40), seed=123).trace.to_jsonl()
            for _ in range(2))
    assert a == b and len(a) > 10_000
