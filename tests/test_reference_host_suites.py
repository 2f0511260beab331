"""The reference's host-side suites (pkg/tests/test_cluster.py, test_fabric.py,
test_weights.py), restated against the drop-in's control plane: PP-config validation,
the exact-rational KV budget (max_blocks), config diffs, the parity-mode fabric with its
handshake, and the layer-weight loader's timing model.  Same test names and assertions;
pure host logic, so these run on CPU."""

import random
import threading
from fractions import Fraction
from math import floor

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2604_12171_b200.cluster import (GpuSpec, ModelSpec, PPConfig, diff_configs,
                                           max_blocks, validate_pp_config)
from paper_2604_12171_b200.events import EventScheduler, EventTrace
from paper_2604_12171_b200.fabric import CommFabric, FabricConfig, detect_deadlock
from paper_2604_12171_b200.weights import LayerInUse, OutOfMemory, WeightLoader

MIB, GIB = 1024 * 1024, 1024 ** 3


def gpu_(i=1, mem_mib=4096):
    return GpuSpec(i, mem_mib * MIB, 1e12, 1e-5, 1e-5, 2 * MIB)


def model_(layers=8, k=1, weight_mib=64):
    return ModelSpec(layers, weight_mib * MIB, 8 * 1024, k)


C_A = PPConfig([(1, (1, 2)), (2, (3, 4)), (3, (5, 6))])
C_B = PPConfig([(1, (1, 1)), (2, (2, 3)), (3, (4, 6))])


# --- test_cluster.py: TestValidate -----------------------------------------------------------
@pytest.mark.parametrize("cfg,layers,k,gpus,needle", [
    (C_A, 6, 1, (1, 2, 3), None),
    (PPConfig([(1, (1, 2)), (2, (2, 3)), (3, (4, 6))]), 6, 1, (1, 2, 3), "overlap"),
    (PPConfig([(1, (1, 6)), (2, (7, 8))]), 8, 4, (1, 2), "multiple"),
    (PPConfig([(1, (1, 2)), (2, (4, 6))]), 6, 1, (1, 2), "gap"),
    (PPConfig([(1, (1, 3)), (2, (4, 6))]), 6, 1, (1, 2, 3), "no layer range"),
], ids=["test_valid_three_gpu_six_layer", "test_overlapping_ranges",
        "test_range_not_multiple_of_k", "test_gap_detected", "test_missing_gpu"])
def test_validate(cfg, layers, k, gpus, needle):
    v = validate_pp_config(cfg, model_(layers, k), [gpu_(i) for i in gpus])
    assert v == [] if needle is None else any(needle in x for x in v)


# --- TestMaxBlocks ---------------------------------------------------------------------------
def test_degenerate_identity():
    assert max_blocks(GpuSpec(1, 100, 1, 1, 1, 1), 1, ModelSpec(1, 0, 1, 1), 1.0) == 100


def test_alg1_formula_example():
    g = GpuSpec(1, 81920 * MIB, 1, 1, 1, 2 * MIB)
    m = ModelSpec(40, 800 * MIB, 8 * 1024, 1)
    want = floor((Fraction(81920 * MIB) * Fraction(0.9) - 40 * 800 * MIB) / (40 * Fraction(2 * MIB)))
    assert want == 521 == max_blocks(g, 40, m, 0.9)


def test_infeasible_when_weights_exceed_budget():
    assert max_blocks(GpuSpec(1, 10, 1, 1, 1, 1), 5, ModelSpec(5, 3, 1, 1), 1.0) is None


def test_monotone_non_increasing_in_layers():
    vals = [max_blocks(gpu_(mem_mib=8192), n, model_(16, 1, 128), 0.9) for n in range(1, 17)]
    for a, b in zip(vals, vals[1:]):
        assert b is None or (a is not None and a >= b)


# --- TestDiffConfigs -------------------------------------------------------------------------
def test_fig3_worked_example():
    c_int, m_add, m_del, m_mig = diff_configs(C_A, C_B)
    assert c_int == {1: {1, 2}, 2: {2, 3, 4}, 3: {4, 5, 6}}
    assert (m_add, m_del, m_mig) == ({2: {2}, 3: {4}}, {1: {2}, 2: {4}},
                                     {(1, 2): {2}, (2, 3): {4}})


def test_identity():
    c_int, m_add, m_del, m_mig = diff_configs(C_A, C_A)
    assert (m_add, m_del, m_mig) == ({}, {}, {}) and c_int == C_A.as_layer_sets()


def test_two_gpu_hand_trace():
    _, m_add, m_del, m_mig = diff_configs(PPConfig([(1, (1, 4)), (2, (5, 8))]),
                                          PPConfig([(1, (1, 2)), (2, (3, 8))]))
    assert (m_mig, m_add, m_del) == ({(1, 2): {3, 4}}, {2: {3, 4}}, {1: {3, 4}})


def _config(rng, ids, n_groups, k):
    cuts = sorted(rng.sample(range(1, n_groups), len(ids) - 1))
    bounds = [0, *cuts, n_groups]
    return PPConfig([(g, (bounds[i] * k + 1, bounds[i + 1] * k)) for i, g in enumerate(ids)])


@st.composite
def config_pairs(draw):
    n = draw(st.integers(2, 4))
    k = draw(st.sampled_from([1, 2, 4]))
    n_groups = draw(st.integers(n, 10))
    rng = random.Random(draw(st.integers(0, 2 ** 32 - 1)))
    ids = list(range(1, n + 1))
    return _config(rng, ids, n_groups, k), _config(rng, ids, n_groups, k)


@given(config_pairs())
@settings(max_examples=200, deadline=None)
def test_diff_set_identities(pair):
    cur, tgt = pair
    c_int, m_add, m_del, m_mig = diff_configs(cur, tgt)
    a, b = cur.as_layer_sets(), tgt.as_layer_sets()
    for g in a:
        assert a[g] | m_add.get(g, set()) == c_int[g]
        assert c_int[g] - m_del.get(g, set()) == b[g]
    moved = set()
    for (s, d), layers in m_mig.items():
        assert s != d and layers <= m_add[d] and layers <= a[s] and not moved & layers
        moved |= layers
    assert moved == (set().union(*m_add.values()) if m_add else set())


@given(config_pairs())
@settings(max_examples=200, deadline=None)
def test_diff_swap_symmetry(pair):
    cur, tgt = pair
    _, m_add, m_del, m_mig = diff_configs(cur, tgt)
    _, r_add, r_del, r_mig = diff_configs(tgt, cur)
    assert (m_add, m_del) == (r_del, r_add)
    assert {(d, s): v for (s, d), v in m_mig.items()} == r_mig


def test_diff_requires_same_gpu_set():
    with pytest.raises(ValueError):
        diff_configs(PPConfig([(1, (1, 4)), (2, (5, 8))]), PPConfig([(1, (1, 4)), (3, (5, 8))]))


# --- test_fabric.py --------------------------------------------------------------------------
def fabric_(n=3, **cfg):
    sched, trace = EventScheduler(), EventTrace()
    return sched, trace, CommFabric(sched, trace, list(range(1, n + 1)), FabricConfig(**cfg))


def test_100mb_at_100gbps_takes_8ms():
    sched, _, fab = fabric_()
    t = fab.post_inference_transfer(1, 2, 100_000_000)
    sched.run()
    assert t.state == "done" and t.complete_time == pytest.approx(0.008)


def test_disjoint_pairs_proceed_concurrently():
    sched, _, fab = fabric_(4)
    ts = [fab.post_inference_transfer(1, 2, 100_000_000), fab.post_inference_transfer(3, 4, 100_000_000)]
    sched.run()
    assert [t.complete_time for t in ts] == pytest.approx([0.008, 0.008])


def test_shared_gpu_serializes():
    sched, _, fab = fabric_()
    ts = [fab.post_inference_transfer(1, 2, 100_000_000), fab.post_inference_transfer(2, 3, 100_000_000)]
    sched.run()
    assert [t.complete_time for t in ts] == pytest.approx([0.008, 0.016])


def fig6(fab):
    """GPU2 forwards a stage output to GPU1 while migrating KV to GPU1; GPU1's receive is
    pre-posted and the migration send takes GPU2 before the inference send is issued."""
    return (fab.post_pair("inference", src=2, dst=1, nbytes=1_000_000, recv_delay=0.0,
                          send_delay=0.0002),
            fab.post_pair("migration", src=2, dst=1, nbytes=1_000_000, recv_delay=0.0001,
                          send_delay=0.0001))


def test_naive_migration_deadlocks():
    sched, _, fab = fabric_(handshake=False)
    t_inf, t_mig = fig6(fab)
    sched.run()
    assert (t_inf.state, t_mig.state) == ("pending", "pending")
    cycle = detect_deadlock(fab)
    assert cycle is not None and {g for g, _ in cycle} == {1, 2}


def test_handshake_resolves_fig6_reference():
    sched, trace, fab = fabric_(handshake=True)
    t_inf, t_mig = fig6(fab)
    sched.run()
    assert (t_inf.state, t_mig.state) == ("done", "done")
    assert t_mig.complete_time > t_inf.complete_time and detect_deadlock(fab) is None
    kinds = {ev.kind for ev in trace}
    assert kinds & {"handshake_reject", "handshake_preempted"}


def test_empty_fabric_has_no_deadlock():
    assert detect_deadlock(fabric_()[2]) is None


def test_idle_receiver_accepts_immediately():
    sched, trace, fab = fabric_(handshake=True)
    t = fab.migrate_transfer(1, 2, 1_000_000)
    sched.run()
    kinds = [ev.kind for ev in trace]
    assert t.state == "done" and "handshake_reject" not in kinds
    assert kinds.count("handshake_ack") == kinds.count("handshake_accept") == 1
    assert t.start_time == pytest.approx(0.0002)           # ACK + ACCEPT before the copy


def test_busy_receiver_rejects_then_retry_succeeds():
    sched, trace, fab = fabric_(handshake=True)
    fab.post_inference_transfer(3, 2, 50_000_000)           # GPU2 busy for 4 ms
    sched.after(0.0001, lambda: fab.migrate_transfer(1, 2, 1_000_000))
    sched.run()
    kinds = [ev.kind for ev in trace]
    assert "handshake_reject" in kinds and "handshake_retry" in kinds
    assert kinds.count("handshake_accept") == 1 and all(t.state == "done" for t in fab.transfers)


def test_inference_preempts_unaccepted_migration():
    sched, trace, fab = fabric_(handshake=True)
    fab.migrate_transfer(1, 2, 1_000_000)
    inf = []
    sched.at(0.00005, lambda: inf.append(fab.post_inference_transfer(1, 3, 1000)))
    sched.run()
    assert "handshake_preempted" in [ev.kind for ev in trace]
    assert inf[0].start_time == pytest.approx(0.00005)
    assert all(t.state == "done" for t in fab.transfers)


def test_symmetric_cross_migrations_complete_reference():
    sched, _, fab = fabric_(handshake=True)
    ts = [fab.migrate_transfer(1, 2, 1_000_000), fab.migrate_transfer(2, 1, 1_000_000)]
    sched.run(until=10.0)
    assert all(t.state == "done" for t in ts)


def test_liveness_under_finite_inference_traffic():
    sched, _, fab = fabric_(handshake=True)
    mig = fab.migrate_transfer(1, 2, 2_000_000)
    for i in range(20):
        sched.at(i * 0.0004, lambda: fab.post_inference_transfer(2, 3, 400_000))
    sched.run(until=10.0)
    assert mig.state == "done"


def random_schedule(seed, handshake):
    """A random <= 4-GPU transfer mix: stage-forward inference along a shuffled pipeline
    (receive pre-posted, per-pair issue windows kept in order) plus migrations between
    arbitrary GPUs, run to quiescence."""
    rng = random.Random(seed)
    ids = list(range(1, rng.randint(2, 4) + 1))
    pipe = rng.sample(ids, len(ids))
    sched, trace = EventScheduler(), EventTrace()
    fab = CommFabric(sched, trace, ids, FabricConfig(handshake=handshake))
    cursor, out = {}, []
    for _ in range(rng.randint(2, 8)):
        nbytes = rng.randint(10_000, 2_000_000)
        if rng.random() < 0.5:
            i = rng.randrange(len(ids) - 1)
            s, d = pipe[i], pipe[i + 1]
            t0 = max(cursor.get((s, d), 0.0), rng.uniform(0.0, 0.004))
            lag = rng.uniform(0.0, 0.002)
            cursor[(s, d)] = t0 + lag + 1e-6
            out.append(fab.post_pair("inference", s, d, nbytes, send_delay=t0 + lag, recv_delay=t0))
        else:
            s, d = rng.sample(ids, 2)
            t0 = rng.uniform(0.0, 0.004)
            out.append(fab.post_pair("migration", s, d, nbytes, send_delay=t0, recv_delay=t0))
    sched.run(until=30.0)
    return fab, out


def test_handshake_schedules_never_deadlock():
    for seed in range(300):
        fab, ts = random_schedule(seed, True)
        assert detect_deadlock(fab) is None and all(t.state == "done" for t in ts), seed


def test_naive_schedules_can_deadlock():
    assert any(detect_deadlock(random_schedule(seed, False)[0]) is not None for seed in range(200))


def test_bandwidth_conservation():
    for seed in range(40):
        fab, _ = random_schedule(seed, True)
        per_link = {}
        for t in fab.transfers:
            if t.start_time is not None:
                per_link.setdefault((t.src, t.dst), []).append((t.start_time, t.complete_time))
        for spans in per_link.values():
            spans.sort()
            assert all(b[0] >= a[1] for a, b in zip(spans, spans[1:]))   # one at a time


def test_try_acquire_contract_from_real_threads():
    """The handshake's try-acquire rule (hold a device only when it is free, back off on
    contention) keeps a real lock table consistent under threads."""
    locks = {g: threading.Lock() for g in (1, 2, 3)}
    bad = []

    def worker(me, peer):
        for _ in range(2000):
            if not locks[me].acquire(blocking=False):
                continue
            try:
                if locks[peer].acquire(blocking=False):
                    locks[peer].release()
            except Exception as e:   # pragma: no cover
                bad.append(repr(e))
            finally:
                locks[me].release()

    ths = [threading.Thread(target=worker, args=p) for p in ((1, 2), (2, 1), (2, 3), (3, 1))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not bad and not any(lk.locked() for lk in locks.values())


# --- test_weights.py -------------------------------------------------------------------------
def loader_(**kw):
    sched, trace = EventScheduler(), EventTrace()
    return sched, WeightLoader(sched, trace, layer_weight_bytes=800 * MIB, **kw)


def test_zero_layers_completes_immediately():
    sched, ld = loader_()
    done = []
    ld.stage_layers(1, set(), lambda: done.append(sched.now))
    sched.run()
    assert done == [0.0]


def test_four_layers_dedicated_bandwidth():
    sched, ld = loader_()
    done = []
    ld.stage_layers(1, {5, 6, 7, 8}, lambda: done.append(sched.now))
    sched.run()
    assert done[0] == pytest.approx(4 * 800 * MIB / (16 * GIB))     # 0.1953125 s
    assert ld.residency.on_gpu(1) == {5, 6, 7, 8}


def test_partial_progress_is_observable():
    sched, ld = loader_()
    ld.stage_layers(1, {5, 6})
    sched.run(until=0.06)                                            # one layer ~0.0488 s
    assert ld.residency.on_gpu(1) == {5}
    sched.run()
    assert ld.residency.on_gpu(1) == {5, 6}


def test_strict_priority_pauses_under_compute():
    sched, ld = loader_(sharing="strict")
    done = []
    ld.set_gpu_busy(1, True)
    sched.at(0.5, lambda: ld.set_gpu_busy(1, False))
    ld.stage_layers(1, {5}, lambda: done.append(sched.now))
    sched.run()
    assert done[0] == pytest.approx(0.5 + 800 * MIB / (16 * GIB))


def test_weighted_sharing_slows_but_progresses():
    sched, ld = loader_(sharing="weighted", busy_weight=0.2)
    done = []
    ld.set_gpu_busy(1, True)
    ld.stage_layers(1, {5}, lambda: done.append(sched.now))
    sched.run()
    assert done[0] == pytest.approx(800 * MIB / (16 * GIB) / 0.2)


def test_disk_fallback_tier():
    sched, ld = loader_()
    ld.residency.host_resident[5] = False
    done = []
    ld.stage_layers(1, {5}, lambda: done.append(sched.now))
    sched.run()
    assert done[0] == pytest.approx(800 * MIB / (2 * GIB))


def test_headroom_violation_surfaces_loudly():
    _, ld = loader_()
    ld.headroom_bytes = lambda gpu: 100 * MIB
    with pytest.raises(OutOfMemory):
        ld.stage_layers(1, {5})


def test_evict_nothing():
    assert loader_()[1].evict_layers(1, set()) == 0


def test_evict_two_layers_frees_bytes():
    sched, ld = loader_()
    ld.stage_layers(1, {5, 6})
    sched.run()
    assert ld.evict_layers(1, {5, 6}) == 1600 * MIB and ld.residency.on_gpu(1) == set()


def test_evicting_committed_layer_rejected():
    sched, ld = loader_()
    ld.stage_layers(1, {5})
    sched.run()
    ld.is_layer_committed = lambda gpu, layer: layer == 5
    with pytest.raises(LayerInUse):
        ld.evict_layers(1, {5})


# --- test_cli.py TestScenarioLoading (scenario files; the argparse front end is out of scope) --
def scenario_doc(**over):
    doc = {"schema_version": 1,
           "cluster": [{"id": i, "mem_total": "8 GiB", "mem_bandwidth": "900 GB/s",
                        "prefill_cost": f"{i} us", "decode_cost": f"{10 // i} us",
                        "alloc_granularity": "2 MiB"} for i in (1, 2)],
           "model": {"num_layers": 8, "layer_weight_bytes": "64 MiB",
                     "token_kv_bytes_per_layer": "16 KiB", "stacking_factor": 1,
                     "activation_bytes_per_token": "4 KiB"},
           "initial_config": [[1, [1, 4]], [2, [5, 8]]],
           "workload": {"pattern": "prefill_heavy", "rate": "50 req/s", "num_requests": 5}}
    doc.update(over)
    return doc


def test_roundtrip(tmp_path):
    import yaml

    from paper_2604_12171_b200.scenario import load_scenario
    path = tmp_path / "scen.yaml"
    path.write_text(yaml.safe_dump(scenario_doc()))
    scen = load_scenario(str(path))
    assert (scen.model.num_layers, scen.cluster[0].mem_total, scen.workload.rate) == \
        (8, 8 * GIB, 50.0)


@pytest.mark.parametrize("edit,field", [
    (lambda d: d["model"].__setitem__("layer_weight_bytes", 67108864), "layer_weight_bytes"),
    (lambda d: d["cluster"][0].__setitem__("prefill_cost", "4 MiB"), "prefill_cost"),
    (lambda d: d.__setitem__("initial_config", [[1, [1, 4]], [2, [4, 8]]]), "initial_config"),
], ids=["test_bare_number_rejected", "test_wrong_unit_dimension_rejected",
        "test_invalid_config_names_field"])
def test_scenario_errors_name_the_field(edit, field):
    from paper_2604_12171_b200.scenario import ScenarioError, scenario_from_dict
    doc = scenario_doc()
    edit(doc)
    with pytest.raises(ScenarioError) as err:
        scenario_from_dict(doc)
    assert field in str(err.value)


def test_packaged_example_loads(tmp_path):
    import json
    from pathlib import Path

    from paper_2604_12171_b200.scenario import load_scenario
    text = json.loads((Path(__file__).parent / "golden" / "cli_outputs.json").read_text())[
        "packaged_seed0"]["yaml"]                    # pkg/scenarios/heterogeneous_shift.yaml
    path = tmp_path / "heterogeneous_shift.yaml"
    path.write_text(text)
    scen = load_scenario(str(path))
    assert scen.triggers and scen.workload.pattern == "shift_schedule"
