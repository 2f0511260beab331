"""CPU tests of the host-side restatement of the reference's control plane: world
model, fabric timing / handshake / deadlock model, event clock, weight staging,
workload and metrics, scenario parsing.  Known answers follow the reference's own
tests (pkg/tests/test_cluster.py, test_fabric.py, test_weights.py, test_cli.py)."""

from fractions import Fraction
from math import floor

import pytest

from paper_2604_12171_b200 import cluster as cl
from paper_2604_12171_b200.engine import (Metrics, WorkloadSpec, compute_metrics,
                                          generate_workload, score)
from paper_2604_12171_b200.events import EventScheduler, EventTrace, stable_hash
from paper_2604_12171_b200.fabric import CommFabric, FabricConfig, detect_deadlock
from paper_2604_12171_b200.scenario import ScenarioError, scenario_from_dict
from paper_2604_12171_b200.weights import GIB, LayerInUse, OutOfMemory, WeightLoader

MIB = 1 << 20


def fabric(n=3, **cfg):
    s, t = EventScheduler(), EventTrace()
    return s, t, CommFabric(s, t, list(range(1, n + 1)), FabricConfig(**cfg))


class TestWorldModel:
    def test_max_blocks_alg1_example_is_521(self):
        gpu = cl.GpuSpec(1, 81920 * MIB, 1, 1, 1, 2 * MIB)
        model = cl.ModelSpec(40, 800 * MIB, 8192, 1)
        want = floor((Fraction(81920 * MIB) * Fraction(0.9) - 40 * 800 * MIB) / (40 * Fraction(2 * MIB)))
        assert want == 521 == cl.max_blocks(gpu, 40, model, 0.9)

    def test_max_blocks_none_when_weights_do_not_fit(self):
        gpu = cl.GpuSpec(1, 10, 1, 1, 1, 1)
        assert cl.max_blocks(gpu, 5, cl.ModelSpec(5, 3, 1, 1), 1.0) is None
        with pytest.raises(ValueError):
            cl.max_blocks(gpu, 0, cl.ModelSpec(5, 3, 1, 1), 1.0)

    def test_fig3_diff(self):
        a = cl.PPConfig([(1, (1, 2)), (2, (3, 4)), (3, (5, 6))])
        b = cl.PPConfig([(1, (1, 1)), (2, (2, 3)), (3, (4, 6))])
        c_int, add, rem, mig = cl.diff_configs(a, b)
        assert c_int == {1: {1, 2}, 2: {2, 3, 4}, 3: {4, 5, 6}}
        assert add == {2: {2}, 3: {4}} and rem == {1: {2}, 2: {4}}
        assert mig == {(1, 2): {2}, (2, 3): {4}}

    def test_validation_messages(self):
        gpus = [cl.GpuSpec(i, 4096 * MIB, 1, 1, 1) for i in (1, 2)]
        model = cl.ModelSpec(8, MIB, 8192, 2)
        assert any("overlap" in v for v in cl.validate_pp_config(
            cl.PPConfig([(1, (1, 4)), (2, (3, 8))]), model, gpus))
        assert any("multiple" in v for v in cl.validate_pp_config(
            cl.PPConfig([(1, (1, 3)), (2, (4, 8))]), model, gpus))
        assert any("gap" in v for v in cl.validate_pp_config(
            cl.PPConfig([(1, (1, 2)), (2, (5, 8))]), model, gpus))
        assert any("no layer range" in v for v in cl.validate_pp_config(
            cl.PPConfig([(1, (1, 8))]), model, gpus))

    def test_enumerate_six_layers_two_gpus(self):
        cfgs = cl.enumerate_pp_configs(6, 1, [1, 2])
        assert [c.range_for(1) for c in cfgs] == [(1, 1), (1, 2), (1, 3), (1, 4), (1, 5)]

    def test_idle_gpu_extension(self):
        gpus = [cl.GpuSpec(i, 4096 * MIB, 1, 1, 1) for i in (1, 2, 3)]
        model = cl.ModelSpec(4, MIB, 8192, 1)
        cur = cl.PPConfig([(1, (1, 2)), (2, (3, 4))])
        tgt = cl.PPConfig([(1, (1, 1)), (2, (2, 3)), (3, (4, 4))])
        assert cl.validate_pp_config(cur, model, gpus, allow_idle_gpus=True) == []
        with pytest.raises(ValueError):
            cl.diff_configs(cur, tgt)
        c_int, add, rem, mig = cl.diff_configs(cur, tgt, True, [1, 2, 3])
        assert c_int[3] == {4} and add == {2: {2}, 3: {4}} and mig == {(1, 2): {2}, (2, 3): {4}}
        assert cl.budget_for(gpus[2], 0, model, 0.9, True) > cl.max_blocks(gpus[0], 1, model, 0.9)


class TestFabricModel:
    def test_100mb_at_100gbps_is_8ms(self):
        s, _, f = fabric()
        t = f.post_inference_transfer(1, 2, 100_000_000)
        s.run()
        assert t.complete_time == pytest.approx(0.008)

    def test_shared_gpu_serialises(self):
        s, _, f = fabric()
        a = f.post_inference_transfer(1, 2, 100_000_000)
        b = f.post_inference_transfer(2, 3, 100_000_000)
        s.run()
        assert (a.complete_time, b.complete_time) == pytest.approx((0.008, 0.016))

    @staticmethod
    def fig6(f):
        ti = f.post_pair("inference", src=2, dst=1, nbytes=1_000_000, recv_delay=0.0,
                         send_delay=0.0002)
        tm = f.post_pair("migration", src=2, dst=1, nbytes=1_000_000, recv_delay=0.0001,
                         send_delay=0.0001)
        return ti, tm

    def test_naive_two_communicators_deadlock(self):
        s, _, f = fabric(handshake=False)
        ti, tm = self.fig6(f)
        s.run()
        assert ti.state == tm.state == "pending"
        assert {g for g, _ in detect_deadlock(f)} == {1, 2}

    def test_handshake_resolves_fig6(self):
        s, t, f = fabric(handshake=True)
        ti, tm = self.fig6(f)
        s.run()
        assert ti.state == tm.state == "done" and tm.complete_time > ti.complete_time
        assert detect_deadlock(f) is None

    def test_idle_receiver_two_control_latencies(self):
        s, t, f = fabric()
        x = f.migrate_transfer(1, 2, 1_000_000)
        s.run()
        assert x.start_time == pytest.approx(2e-4)
        kinds = [e.kind for e in t]
        assert kinds.count("handshake_ack") == kinds.count("handshake_accept") == 1

    def test_symmetric_cross_migrations_complete(self):
        s, _, f = fabric()
        a = f.migrate_transfer(1, 2, 1_000_000)
        b = f.migrate_transfer(2, 1, 1_000_000)
        s.run(until=10.0)
        assert a.state == b.state == "done"


def test_scheduler_ties_fire_in_scheduling_order():
    s = EventScheduler()
    seen = []
    for i in range(5):
        s.at(1.0, lambda i=i: seen.append(i))
    s.at(0.5, lambda: seen.append("first"))
    s.run()
    assert seen == ["first", 0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        s.at(0.1, lambda: None)
    tr = EventTrace()
    tr.emit(1.0, "a", "k", x=1)
    with pytest.raises(ValueError):
        tr.emit(0.5, "a", "k")
    assert tr.to_jsonl() == '{"actor": "a", "kind": "k", "t": 1.0, "x": 1}\n'


class TestWeights:
    def test_strict_staging_pauses_while_busy(self):
        s, t = EventScheduler(), EventTrace()
        w = WeightLoader(s, t, GIB, host_bandwidth=GIB)
        done = []
        w.stage_layers(1, {5, 6}, lambda: done.append(s.now))
        s.at(0.5, lambda: w.set_gpu_busy(1, True))
        s.at(1.5, lambda: w.set_gpu_busy(1, False))
        s.run()
        assert done == [pytest.approx(3.0)]
        assert w.residency.on_gpu(1) == {5, 6}

    def test_evict_committed_layer_rejected_and_headroom(self):
        s, t = EventScheduler(), EventTrace()
        w = WeightLoader(s, t, GIB)
        w.is_layer_committed = lambda gpu, layer: layer == 3
        with pytest.raises(LayerInUse):
            w.evict_layers(1, {3})
        w.headroom_bytes = lambda gpu: GIB // 2
        with pytest.raises(OutOfMemory):
            w.stage_layers(1, {7})


def test_workload_deterministic_and_metrics():
    spec = WorkloadSpec("shift_schedule", rate=5.0, num_requests=20,
                        shifts=((0.0, "prefill_heavy"), (2.0, "decode_heavy")))
    a, b = generate_workload(spec, 3), generate_workload(spec, 3)
    assert [(r.id, r.arrival_time, r.pattern) for r in a] == \
           [(r.id, r.arrival_time, r.pattern) for r in b]
    assert {r.pattern for r in a} == {"prefill_heavy", "decode_heavy"}
    tr = EventTrace()
    tr.emit(0.0, "engine", "request_arrival", id="x", input_len=4, output_len=3, pattern="p")
    tr.emit(1.0, "engine", "first_token", id="x")
    tr.emit(3.0, "engine", "request_done", id="x")
    m = compute_metrics(tr)
    assert (m.ttft_mean, m.tpot_mean, m.completed) == (1.0, 1.0, 1)
    assert score([Metrics(ttft_mean=1), Metrics(ttft_mean=2)])[0] > score(
        [Metrics(ttft_mean=1), Metrics(ttft_mean=2)])[1]


def test_scenario_units_are_mandatory():
    base = {"cluster": [{"id": 1, "mem_total": "80 GiB", "mem_bandwidth": "2039 GB/s",
                         "prefill_cost": "4 us", "decode_cost": "6 us"}],
            "model": {"num_layers": 2, "layer_weight_bytes": "1 GiB",
                      "token_kv_bytes_per_layer": "64 KiB", "stacking_factor": 1},
            "initial_config": [[1, [1, 2]]],
            "workload": {"pattern": "prefill_heavy", "rate": "2 req/s", "num_requests": 3},
            "reconfig_triggers": [{"at": "1 s", "target_config": [[1, [1, 2]]], "tau": "50 tokens"}],
            "fabric": {"link_bandwidth": "100 Gbps"}}
    sc = scenario_from_dict(base)
    assert sc.cluster[0].mem_total == 80 << 30 and sc.fabric.link_bandwidth == 1.25e10
    assert sc.triggers[0].tau == 50 and sc.workload.rate == 2.0
    bad = dict(base)
    bad["cluster"] = [dict(base["cluster"][0], mem_total=80)]
    with pytest.raises(ScenarioError):
        scenario_from_dict(bad)


def test_stable_hash_golden():
    assert stable_hash("r0000", 0) == 4468064692898534167
    assert stable_hash("a", 0, 5) == 7693380175056537723
