"""The reference's coordinator and engine suites (pkg/tests/test_coordinator.py,
pkg/tests/test_engine.py:1-130), restated against the drop-in.  Feasibility and workload
generation are host logic (CPU); every run of a Simulation keeps its KV on the GPU."""

import pytest

MIB, KIB = 1024 * 1024, 1024
gpu = pytest.mark.gpu


def _cl():
    from paper_2604_12171_b200 import cluster
    return cluster


def fig3_gpus(mem_mib=4096):
    c = _cl()
    return {i: c.GpuSpec(i, mem_mib * MIB, 1e12, 1e-6, 1e-5, 2 * MIB) for i in (1, 2, 3)}


def fig3_model():
    return _cl().ModelSpec(6, 64 * MIB, 8 * KIB, 1, 2 * KIB)


def configs():
    c = _cl()
    return (c.PPConfig([(1, (1, 2)), (2, (3, 4)), (3, (5, 6))]),
            c.PPConfig([(1, (1, 1)), (2, (2, 3)), (3, (4, 6))]))


def fig3(triggers=(), num_requests=4, rate=200.0, tau=50):
    from paper_2604_12171_b200.coordinator import FeatureFlags
    from paper_2604_12171_b200.engine import WorkloadSpec
    from paper_2604_12171_b200.scenario import ReconfigTrigger, Scenario
    c_a, _ = configs()
    return Scenario(cluster=list(fig3_gpus().values()), model=fig3_model(), initial_config=c_a,
                    workload=WorkloadSpec(pattern="decode_heavy", rate=rate,
                                          num_requests=num_requests),
                    triggers=[ReconfigTrigger(at, tgt, tau=tau) for at, tgt in triggers],
                    flags=FeatureFlags())


# --- TestFeasibility (test_coordinator.py:32-60) -------------------------------------------
def test_fig3_plan():
    from paper_2604_12171_b200.coordinator import feasibility
    c_a, c_b = configs()
    plan = feasibility(c_a, c_b, fig3_gpus(), fig3_model(), util_ratio=0.9, used_blocks=10)
    assert plan.m_mig == {(1, 2): {2}, (2, 3): {4}}
    assert (plan.m_add, plan.m_del) == ({2: {2}, 3: {4}}, {1: {2}, 2: {4}})
    assert plan.b_shrink <= plan.b_new


def test_noop_plan():
    from paper_2604_12171_b200.coordinator import feasibility
    c_a, _ = configs()
    plan = feasibility(c_a, c_a, fig3_gpus(), fig3_model(), 0.9, 0)
    assert plan.is_noop and plan.m_mig == {}


def test_used_blocks_boundary():
    from paper_2604_12171_b200.coordinator import Infeasible, feasibility
    c_a, c_b = configs()
    gpus, model = fig3_gpus(), fig3_model()
    budget = feasibility(c_a, c_b, gpus, model, 0.9, 0).b_shrink
    feasibility(c_a, c_b, gpus, model, 0.9, budget)          # exactly at the budget: ok
    with pytest.raises(Infeasible):
        feasibility(c_a, c_b, gpus, model, 0.9, budget + 1)  # one block over: abort


def test_weights_that_cannot_fit():
    from paper_2604_12171_b200.coordinator import Infeasible, feasibility
    c_a, c_b = configs()
    with pytest.raises(Infeasible):
        feasibility(c_a, c_b, fig3_gpus(mem_mib=512), _cl().ModelSpec(6, 200 * MIB, 8 * KIB, 1),
                    0.9, 0)


# --- TestReconfigureNoop / TestReconfigureFig3 (test_coordinator.py:75-173) -----------------
@gpu
def test_noop_success_zero_pause_state_identical():
    from paper_2604_12171_b200.simulation import Simulation
    c_a, _ = configs()
    sim = Simulation(fig3(num_requests=0))
    before = sim.state_digest()
    done = []
    sim.coordinator.reconfigure(sim.coordinator.feasibility(c_a), done.append)
    sim.scheduler.run()
    assert done[0].outcome == "success" and done[0].pause_duration == 0.0
    assert sim.state_digest() == before


@pytest.fixture(scope="module")
def fig3_run():
    from paper_2604_12171_b200.simulation import Simulation
    _, c_b = configs()
    sim = Simulation(fig3(triggers=[(0.02, c_b)], num_requests=4, rate=500.0), seed=5)
    return sim, sim.run()


@gpu
def test_success_and_committed_config(fig3_run):
    sim, res = fig3_run
    assert [s.outcome for s in sim.statuses] == ["success"]
    assert sim.engine.committed_config == configs()[1] and res.metrics.completed == 4


@gpu
def test_phase_ordering_matches_dependency_dag(fig3_run):
    ts = fig3_run[0].statuses[0].timestamps
    assert ts["resize_end"] <= min(ts["weightload_start"], ts["migration_start"])
    assert ts["commit_start"] >= max(ts["convergence_time"], ts["weightload_end"])


@gpu
def test_primitive_names_recorded(fig3_run):
    names = {ev.payload["name"] for ev in fig3_run[1].trace if ev.kind == "primitive"}
    assert {"CompactKV", "ResizeKV", "AddLayerWeights", "StartKVMigration",
            "SyncAndCommit"} <= names


@gpu
def test_migration_consistency_at_commit(fig3_run):
    sim, _ = fig3_run
    st = sim.statuses[0]
    assert st.source_snapshots
    for (src, dst), groups in st.migrated_groups.items():
        for g in groups:
            have = sim.stores[dst].snapshot_group(g)
            for req, fps in st.source_snapshots[(src, dst)][g].items():
                assert have.get(req, ())[:len(fps)] == fps


@gpu
def test_atomic_commit_no_mixed_microbatch(fig3_run):
    trace = fig3_run[1].trace
    resume = next(ev.time for ev in trace if ev.kind == "commit_pause_end")
    spans = {}
    for ev in trace:
        if ev.kind in ("stage_start", "stage_end"):
            spans.setdefault(ev.payload["mb"], []).append(ev.time)
    for times in spans.values():
        assert max(times) <= resume or min(times) >= resume


@gpu
def test_obsolete_state_deleted(fig3_run):
    sim, _ = fig3_run
    on = sim.loader.residency.on_gpu
    assert 2 not in on(1) and 4 not in on(2)
    assert 1 not in sim.stores[1].resident_groups      # layer 2's group (k = 1)
    assert (on(2), on(3)) == ({2, 3}, {4, 5, 6})


@gpu
def test_infeasible_trigger_recorded_not_crash():
    from paper_2604_12171_b200.engine import WorkloadSpec
    from paper_2604_12171_b200.scenario import ReconfigTrigger, Scenario
    from paper_2604_12171_b200.simulation import Simulation
    c = _cl()
    c_a, _ = configs()
    scen = Scenario(cluster=list(fig3_gpus(mem_mib=768).values()),
                    model=c.ModelSpec(6, 200 * MIB, 8 * KIB, 1, 2 * KIB), initial_config=c_a,
                    workload=WorkloadSpec("prefill_heavy", rate=100.0, num_requests=1),
                    triggers=[ReconfigTrigger(0.001, c.PPConfig([(1, (1, 4)), (2, (5, 5)),
                                                                  (3, (6, 6))]))])
    sim = Simulation(scen, seed=1)
    res = sim.run()
    ends = [ev for ev in res.trace if ev.kind == "reconfigure_end"]
    assert ends and ends[0].payload["outcome"] == "infeasible"
    assert sim.engine.committed_config == c_a and res.metrics.reconfig_outcome == "infeasible"


# --- test_engine.py:18-130 -----------------------------------------------------------------
def tiny(num_requests=3, rate=100.0, n_gpus=1, layers=4, pattern="prefill_heavy", max_batch=32):
    from paper_2604_12171_b200.engine import WorkloadSpec
    from paper_2604_12171_b200.scenario import Scenario
    c = _cl()
    per = layers // n_gpus
    return Scenario(
        cluster=[c.GpuSpec(i, 2048 * MIB, 1e12, 1e-6, 1e-5, 2 * MIB) for i in range(1, n_gpus + 1)],
        model=c.ModelSpec(layers, 16 * MIB, 8 * KIB, 1, 2 * KIB),
        initial_config=c.PPConfig([(i, ((i - 1) * per + 1, i * per)) for i in range(1, n_gpus + 1)]),
        workload=WorkloadSpec(pattern=pattern, rate=rate, num_requests=num_requests),
        triggers=[], max_batch=max_batch)


def test_exact_counts_and_means():
    from paper_2604_12171_b200.engine import WorkloadSpec, generate_workload
    reqs = generate_workload(WorkloadSpec("prefill_heavy", rate=2.0, num_requests=200), seed=7)
    assert len(reqs) == 200
    assert (sum(r.input_len for r in reqs) / 200, sum(r.output_len for r in reqs) / 200) == (512, 16)


def test_jitter_keeps_means_close():
    from paper_2604_12171_b200.engine import WorkloadSpec, generate_workload
    reqs = generate_workload(WorkloadSpec("decode_heavy", rate=2.0, num_requests=400, jitter=True),
                             seed=7)
    assert 128 * 0.9 < sum(r.input_len for r in reqs) / len(reqs) < 128 * 1.1


def test_same_seed_identical():
    from paper_2604_12171_b200.engine import WorkloadSpec, generate_workload
    spec = WorkloadSpec("decode_heavy", rate=3.0, num_requests=50)
    a, b = (generate_workload(spec, seed=11) for _ in range(2))
    assert [(r.arrival_time, r.input_len) for r in a] == [(r.arrival_time, r.input_len) for r in b]


def test_huge_rate_bursts():
    from paper_2604_12171_b200.engine import WorkloadSpec, generate_workload
    reqs = generate_workload(WorkloadSpec("prefill_heavy", rate=1e9, num_requests=20), seed=1)
    assert reqs[-1].arrival_time < 1e-6


def test_shift_schedule_switches_pattern():
    from paper_2604_12171_b200.engine import WorkloadSpec, generate_workload
    reqs = generate_workload(WorkloadSpec("shift_schedule", rate=1.0, num_requests=100,
                                          shifts=((0.0, "prefill_heavy"), (50.0, "decode_heavy"))),
                             seed=3)
    assert all((r.pattern == "prefill_heavy") == (r.arrival_time < 50.0) for r in reqs)


@gpu
def test_ttft_and_tpot():
    from paper_2604_12171_b200.simulation import run_scenario
    m = run_scenario(tiny(num_requests=1, rate=1e6), seed=0).metrics
    # one GPU, 4 layers: TTFT = prefill_cost x layers x input, TPOT = one decode step
    assert m.ttft_mean == pytest.approx(1e-6 * 4 * 512)
    assert m.tpot_mean == pytest.approx(1e-5 * 4) and m.completed == 1


@gpu
def test_pipeline_order_invariant():
    from paper_2604_12171_b200.simulation import run_scenario
    res = run_scenario(tiny(num_requests=4, n_gpus=2, rate=1000.0), seed=1)
    spans = {}
    for ev in res.trace:
        if ev.kind in ("stage_start", "stage_end"):
            st = spans.setdefault(ev.payload["mb"], {}).setdefault(ev.payload["stage"], [0.0, 0.0])
            st[ev.kind == "stage_end"] = ev.time
    for stages in spans.values():
        order = sorted(stages)
        for a, b in zip(order, order[1:]):
            assert stages[b][0] >= stages[a][1]      # stage i+1 starts after stage i ends


@gpu
def test_token_conservation():
    from paper_2604_12171_b200.simulation import Simulation
    scen = tiny(num_requests=3, rate=50.0, n_gpus=2)
    res = Simulation(scen, seed=2).run()
    arrivals = {e.payload["id"]: e.payload for e in res.trace if e.kind == "request_arrival"}
    n_groups = scen.model.num_layers // scen.model.stacking_factor
    freed = [e for e in res.trace if e.kind == "request_kv_freed"]
    assert freed
    for ev in freed:
        a = arrivals[ev.payload["id"]]
        assert ev.payload["consumed"] == (a["input_len"] + a["output_len"]) * n_groups


@gpu
def test_same_seed_byte_identical_traces():
    from paper_2604_12171_b200.simulation import run_scenario
    a, b = (run_scenario(tiny(num_requests=6, n_gpus=2), seed=9).trace.to_jsonl() for _ in range(2))
    assert a == b


@gpu
def test_different_seed_differs():
    from paper_2604_12171_b200.simulation import run_scenario
    assert run_scenario(tiny(num_requests=6), seed=1).trace.to_jsonl() != \
        run_scenario(tiny(num_requests=6), seed=2).trace.to_jsonl()


# --- TestComputeMetrics / TestScore / TestContinuousBatching (test_engine.py:133-216) -------
def _trace(events):
    from paper_2604_12171_b200.events import EventTrace
    tr = EventTrace()
    for t, kind, payload in events:
        tr.emit(t, "engine", kind, **payload)
    return tr


def _req(rid, n_in, n_out, t_first, t_done):
    return [(0.0, "request_arrival", {"id": rid, "input_len": n_in, "output_len": n_out}),
            (t_first, "first_token", {"id": rid}), (t_done, "request_done", {"id": rid})]


def test_arithmetic_example():
    from paper_2604_12171_b200.engine import compute_metrics
    m = compute_metrics(_trace(_req("r", 100, 17, 2.0, 10.0)))
    assert m.ttft_mean == 2.0 and m.tpot_mean == pytest.approx(0.5)   # 8 s / 16 tokens


def test_output_len_1_excluded_from_tpot():
    from paper_2604_12171_b200.engine import compute_metrics
    assert compute_metrics(_trace(_req("a", 8, 1, 1.0, 1.0))).tpot_mean == 0.0


def test_no_reconfig_means_zero_stop_time():
    from paper_2604_12171_b200.engine import compute_metrics
    m = compute_metrics(_trace(_req("a", 8, 4, 1.0, 2.0)))
    assert (m.stop_time, m.migration_time) == (0.0, 0.0)


def _rows(vals):
    from paper_2604_12171_b200.engine import Metrics
    out = []
    for ttft, tpot, tput in vals:
        m = Metrics()
        m.ttft_mean, m.tpot_mean, m.throughput = ttft, tpot, tput
        out.append(m)
    return out


@pytest.mark.parametrize("vals,want", [
    ([(1.0, 1.0, 10.0), (2.0, 2.0, 5.0)], [1.0, 0.0]),
    ([(1.0, 3.0, 10.0), (1.0, 4.0, 20.0)], [2.0 / 3, 2.0 / 3]),   # tied ttft counts 1 for both
    ([(1.0, 1.0, 1.0)] * 3, [1.0, 1.0, 1.0]),
], ids=["test_best_row_scores_1", "test_degenerate_metric_scores_1_for_all",
        "test_all_identical_rows"])
def test_score(vals, want):
    from paper_2604_12171_b200.engine import score
    assert score(_rows(vals)) == pytest.approx(want)


@gpu
@pytest.mark.parametrize("n,max_batch", [(4, 4), (6, 2)],
                         ids=["test_decode_rounds_batch_requests", "test_max_batch_respected"])
def test_continuous_batching(n, max_batch):
    from paper_2604_12171_b200.simulation import run_scenario
    res = run_scenario(tiny(num_requests=n, rate=1e5, pattern="decode_heavy", max_batch=max_batch),
                       seed=3)
    sizes = [e.payload["batch"] for e in res.trace
             if e.kind == "stage_start" and e.payload["mb_kind"] == "decode"]
    assert 1 < max(sizes) <= max_batch
