"""Switch-point parity: full reconfiguration runs in parity mode (reference event
clock, GPU data plane) must reproduce the reference's own runs bit for bit --
trace bytes (sha256), convergence/commit timestamps, the micro-batch count at
the switch, pause, lags, capacities, metrics and the final state digest.
Mirrors pkg/tests/test_coordinator.py and acceptance criteria 4/6/10."""

import hashlib

import pytest

import sim_scenarios

pytestmark = pytest.mark.gpu


def _run(name):
    from paper_2604_12171_b200.engine import compute_metrics
    from paper_2604_12171_b200.simulation import RunResult, Simulation

    scen, seed, fill = sim_scenarios.golden_runs()[name]
    sim = Simulation(scen, seed=seed)
    if fill:
        fill(sim)
    sim.scheduler.run(until=600.0)
    return sim, RunResult(sim.trace, compute_metrics(sim.trace), sim.statuses, seed)


@pytest.mark.parametrize("name", ["fig3_seed5", "fig3_nopatch", "stoptime_L4", "stoptime_L8",
                                  "hetero_c10_seed123", "hetero_n60_seed7",
                                  "packaged_yaml_seed0"])
def test_run_matches_reference(golden, name):
    want = golden("simulations.json")[name]
    sim, res = _run(name)
    jsonl = res.trace.to_jsonl()
    assert len(res.trace) == want["n_events"]
    assert hashlib.sha256(jsonl.encode()).hexdigest() == want["trace_sha"]
    assert len(sim.statuses) == len(want["statuses"])
    for got, exp in zip(sim.statuses, want["statuses"]):
        assert got.outcome == exp["outcome"]
        assert got.timestamps == exp["timestamps"]          # incl. convergence_time / commit_start
        assert got.pause_duration == exp["pause"]
        assert {str(k): v for k, v in got.lag_at_final_sync.items()} == exp["lag_at_final_sync"]
        assert got.steps_at_commit == want["steps_at_commit"]  # the switch iteration
        # criterion 4 at the commit snapshot
        for pair, groups in got.migrated_groups.items():
            for g in groups:
                assert got.dest_snapshots[pair][g] == got.source_snapshots[pair][g]
    assert {str(g): s.capacity_blocks for g, s in sim.stores.items()} == want["capacities"]
    assert res.metrics.as_row() == want["metrics"]
    assert sim.state_digest() == want["state_digest"]


def test_fig3_structure():
    """pkg/tests/test_coordinator.py:97-173 on the GPU data plane"""
    from paper_2604_12171_b200.cluster import max_blocks

    sim, res = _run("fig3_seed5")
    status = sim.statuses[0]
    assert status.outcome == "success" and sim.engine.committed_config == sim_scenarios.C_B
    resized = {ev.actor for ev in res.trace if ev.kind == "primitive"
               and ev.payload["name"] == "ResizeKV"}
    assert resized == {"gpu1", "gpu2", "gpu3"}
    ts = status.timestamps
    assert ts["resize_end"] <= ts["weightload_start"] <= ts["commit_start"]
    assert ts["commit_start"] >= ts["convergence_time"]
    assert all(lag < 50 for lag in status.lag_at_final_sync.values())
    assert 1 not in sim.stores[1].resident_groups
    assert sim.loader.residency.on_gpu(2) == {2, 3}
    b_new = min(max_blocks(sim_scenarios.fig3_cluster()[g], len(sim_scenarios.C_B.layers_for(g)),
                           sim_scenarios.fig3_model(), 0.9) for g in (1, 2, 3))
    assert all(s.capacity_blocks == b_new for s in sim.stores.values())


def test_rollback_restores_state_bit_exact():
    """pkg/tests/test_coordinator.py:176-201: destination overflow -> rollback"""
    from paper_2604_12171_b200.events import stable_hash
    from paper_2604_12171_b200.simulation import Simulation

    sim = Simulation(sim_scenarios.fig3_scenario(num_requests=0), seed=0)
    s = sim.stores[2].tokens_per_block
    ghost = 40 * s
    for g in (sim.model.group_of(3), sim.model.group_of(4)):
        sim.stores[2].append("ghost", g, ghost, [stable_hash("ghost", g, i) for i in range(ghost)])
    plan = sim.coordinator.feasibility(sim_scenarios.C_B, tau=50)
    for i in range(plan.b_shrink - 22):
        g = sim.model.group_of(5)
        sim.stores[3].append(f"filler{i:03d}", g, s, [stable_hash("filler", i, j) for j in range(s)])
    before = sim.state_digest()
    done = []
    sim.coordinator.reconfigure(plan, done.append)
    sim.scheduler.run()
    assert done[0].outcome == "failed(MigrationOverflow)"
    assert sim.engine.committed_config == sim_scenarios.C_A
    assert sim.state_digest() == before


@pytest.mark.parametrize("name", ["config0_tiny", "config1_8b", "config2_70b", "config3_uneven"])
def test_baseline_config_matches_reference_with_extension(golden, name):
    """BASELINE configs 0-3 (PP 2->3, 2->4, 4->8 with a near-full HBM, uneven 8-GPU re-split)
    against the reference run with the same idle-GPU extension (tests/golden/make_golden.py)."""
    from paper_2604_12171_b200.engine import compute_metrics
    from paper_2604_12171_b200.simulation import Simulation

    want = golden("config_runs.json")[name]
    scen, seed, fill = sim_scenarios.config_runs()[name]
    sim = Simulation(scen, seed=seed)
    if fill:
        fill(sim)
    sim.scheduler.run(until=600.0)
    jsonl = sim.trace.to_jsonl()
    assert len(sim.trace) == want["n_events"]
    assert hashlib.sha256(jsonl.encode()).hexdigest() == want["trace_sha"]
    for got, exp in zip(sim.statuses, want["statuses"]):
        assert got.outcome == exp["outcome"] == "success"
        assert got.timestamps == exp["timestamps"]
        assert got.pause_duration == exp["pause"]
        assert got.steps_at_commit == want["steps_at_commit"]
        for pair, groups in got.migrated_groups.items():
            for g in groups:
                assert got.dest_snapshots[pair][g] == got.source_snapshots[pair][g]
    assert {str(g): s.capacity_blocks for g, s in sim.stores.items()} == want["capacities"]
    assert compute_metrics(sim.trace).as_row() == want["metrics"]
    assert sim.state_digest() == want["state_digest"]


def test_acceptance_criterion_6_stop_time_ablation():
    """Acceptance criterion 6 (pkg/tests/test_acceptance.py:203-248) on the GPU data plane:
    with KV patching the pause stays flat in the number of migrated layers and within the
    analytic bound (residual < tau cells + control overhead); stop-and-copy pauses grow
    with the layer count and exceed the patching pauses tenfold."""
    from paper_2604_12171_b200 import FeatureFlags
    from paper_2604_12171_b200.simulation import Simulation

    tau = 50
    patch, copy = {}, {}
    for n in (4, 8, 12):
        for flags, out in ((None, patch), (FeatureFlags(kv_patch=False, async_weights=False), copy)):
            scen, fill = sim_scenarios.stoptime_scenario(migrate_layers=n, flags=flags)
            sim = Simulation(scen, seed=0)
            fill(sim)
            sim.scheduler.run(until=600.0)
            assert sim.statuses[0].outcome == "success"
            out[n] = sim.statuses[0].pause_duration
    for n in (4, 8, 12):
        assert copy[n] >= 10 * patch[n]
    assert copy[12] > copy[8] > copy[4]
    assert max(patch.values()) / min(patch.values()) < 2.0
    scen, _ = sim_scenarios.stoptime_scenario()
    for n, pause in patch.items():
        bound = tau * scen.model.token_kv_bytes_per_layer * n / scen.fabric.link_bandwidth \
            + 8 * scen.fabric.control_latency
        assert pause <= bound


def test_acceptance_criterion_4_randomized_reconfigurations(golden):
    """Acceptance criterion 4 (pkg/tests/test_acceptance.py:153-182) on the GPU data plane,
    pinned run by run to the reference: 100 randomized reconfigurations (2-4 GPUs, 8-32
    layers) reproduce the reference's trace sha256; every committed one has a bit-exact
    destination KV at the commit snapshot and lag under tau."""
    import time

    from paper_2604_12171_b200.simulation import Simulation

    want = golden("e2e_runs.json")
    t0 = time.time()
    committed = 0
    for seed in range(100):
        scen = sim_scenarios.random_e2e_scenario(seed)
        sim = Simulation(scen, seed=seed)
        sim.scheduler.run(until=60.0)
        sha = hashlib.sha256(sim.trace.to_jsonl().encode()).hexdigest()
        assert sha == want[str(seed)]["trace_sha"], seed
        assert [s.outcome for s in sim.statuses] == want[str(seed)]["outcomes"], seed
        if not sim.statuses or sim.statuses[0].outcome != "success":
            continue
        committed += 1
        st = sim.statuses[0]
        for pair, groups in st.migrated_groups.items():
            for g in groups:
                assert st.dest_snapshots[pair][g] == st.source_snapshots[pair][g], (seed, pair, g)
        for lag in st.lag_at_final_sync.values():
            assert lag < scen.triggers[0].tau
    assert committed >= 60
    assert time.time() - t0 < 120.0


@pytest.mark.parametrize("name,source", [("fig3_seed5", "golden"), ("hetero_c10_seed123", "golden"),
                                         ("config0_tiny", "config")])
def test_parity_run_with_full_4096_byte_cells(golden, monkeypatch, name, source):
    """The parity runs above store a 64-B prefix of each cell (kvstore.DEFAULT_CELL_BYTES)
    so simulated 80 GiB GPUs fit on one B200.  Here the same runs move real 4096-B cells:
    the trace sha256, timestamps and switch point are unchanged, and at the commit (after
    the final sync, before the barrier) every written position of every migrated group on
    every destination equals the source byte for byte -- fingerprint and all k x 4096 B --
    as it does after every patch the receiver applies, and every live cell of every store
    equals the expansion of its fingerprint."""
    from paper_2604_12171_b200 import coordinator, migrator
    from paper_2604_12171_b200.simulation import Simulation

    if source == "golden":
        want = golden("simulations.json")[name]
        scen, seed, fill = sim_scenarios.golden_runs()[name]
    else:
        want = golden("config_runs.json")[name]
        scen, seed, fill = sim_scenarios.config_runs()[name]
    checks = []
    barrier = coordinator.Coordinator._barrier

    def checked_barrier(self, plan, status, pause_start, finish):
        for (src, dst), groups in status.migrated_groups.items():
            rids = sorted({r for g in groups for r in status.source_snapshots[(src, dst)][g]})
            c = self.stores[src].compare_cells(self.stores[dst], groups, rids)
            # every snapshotted position x k layers was compared
            c["expected"] = self.model.stacking_factor * sum(
                len(v) for g in groups for v in status.source_snapshots[(src, dst)][g].values())
            checks.append(("compare", src, dst, c))
        for gpu, st in sorted(self.stores.items()):
            checks.append(("verify", gpu, None, st.verify_cells()))
        return barrier(self, plan, status, pause_start, finish)

    monkeypatch.setattr(coordinator.Coordinator, "_barrier", checked_barrier)
    # and after every patch the receiver applies: the destination's written prefix of every
    # (request, group) of the pair equals the source's, byte for byte
    apply_device = migrator.MigrationStream._apply_device

    def checked_apply(self, dst_store, stale_rids):
        apply_device(self, dst_store, stale_rids)
        src_store = sim.stores[self.src]
        rids = [r for r in dst_store.tables if r in src_store.tables and r not in stale_rids]
        c = src_store.compare_cells(dst_store, sorted(self.groups), rids)
        checks.append(("apply", self.src, self.dst, c))

    monkeypatch.setattr(migrator.MigrationStream, "_apply_device", checked_apply)
    sim = Simulation(scen, seed=seed, cell_bytes=4096)
    assert all(st.cell_bytes == 4096 for st in sim.stores.values())
    if fill:
        fill(sim)
    sim.scheduler.run(until=600.0)
    assert hashlib.sha256(sim.trace.to_jsonl().encode()).hexdigest() == want["trace_sha"]
    assert [s.steps_at_commit for s in sim.statuses][:1] == [want["steps_at_commit"]]
    for got, exp in zip(sim.statuses, want["statuses"]):
        assert got.timestamps == exp["timestamps"]
    assert sim.state_digest() == want["state_digest"]
    compared = [c for kind, _, _, c in checks if kind == "compare"]
    assert compared and all(c["bad_positions"] == 0 and c["missing"] == 0 for c in compared)
    assert all(c["cells"] == c["expected"] for c in compared)
    applied = [c for kind, _, _, c in checks if kind == "apply"]
    assert applied and all(c["bad_positions"] == 0 and c["missing"] == 0 for c in applied)
    assert sum(c["cells"] for c in applied) > 0   # every patch of the run, 4096-B cells
    for kind, gpu, _, v in checks:
        if kind == "verify":
            assert v["bad_bytes"] == 0 and v["first_bad"] == -1, (gpu, v)
    for st in sim.stores.values():   # and at the end of the run
        v = st.verify_cells()
        assert v["bad_bytes"] == 0, v
