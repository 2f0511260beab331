"""Scenario builders with the same parameters as the reference's test scenarios
(pkg/tests/scenarios.py:136-196, pkg/tests/test_coordinator.py:14-73), built on
this package's classes so the golden simulations can be replayed on the GPU box
where the reference does not exist."""

from __future__ import annotations

from paper_2604_12171_b200 import FeatureFlags, GpuSpec, ModelSpec, PPConfig, WorkloadSpec
from paper_2604_12171_b200.scenario import ReconfigTrigger, Scenario

GIB, MIB, KIB = 1024 ** 3, 1024 ** 2, 1024

C_A = PPConfig([(1, (1, 2)), (2, (3, 4)), (3, (5, 6))])
C_B = PPConfig([(1, (1, 1)), (2, (2, 3)), (3, (4, 6))])


def _two_gpus():
    return [GpuSpec(id=1, mem_total=80 * GIB, mem_bandwidth=2.039e12, prefill_cost=4e-6,
                    decode_cost=6e-6),
            GpuSpec(id=2, mem_total=48 * GIB, mem_bandwidth=8.64e11, prefill_cost=1.5e-6,
                    decode_cost=2.4e-5)]


def hetero_scenario(rate=7.0, n=120, k=2, triggers=True, flags=None, tau=50) -> Scenario:
    shift = n / rate / 2
    model = ModelSpec(num_layers=16, layer_weight_bytes=int(2.5 * GIB),
                      token_kv_bytes_per_layer=128 * KIB, stacking_factor=k,
                      activation_bytes_per_token=32 * KIB)
    wl = WorkloadSpec("shift_schedule", rate=rate, num_requests=n,
                      shifts=((0.0, "prefill_heavy"), (shift, "decode_heavy")))
    tgt = PPConfig([(1, (1, 14)), (2, (15, 16))])
    return Scenario(cluster=_two_gpus(), model=model,
                    initial_config=PPConfig([(1, (1, 2)), (2, (3, 16))]), workload=wl,
                    triggers=[ReconfigTrigger(at=shift, target=tgt, tau=tau)] if triggers else [],
                    flags=flags or FeatureFlags())


def stoptime_scenario(migrate_layers=4, flags=None, ghost_tokens=6000):
    model = ModelSpec(num_layers=16, layer_weight_bytes=int(2.5 * GIB),
                      token_kv_bytes_per_layer=64 * KIB, stacking_factor=2,
                      activation_bytes_per_token=32 * KIB)
    edge = 2 + migrate_layers
    scen = Scenario(cluster=_two_gpus(), model=model,
                    initial_config=PPConfig([(1, (1, 2)), (2, (3, 16))]),
                    workload=WorkloadSpec("prefill_heavy", rate=1.0, num_requests=0),
                    triggers=[ReconfigTrigger(at=0.001,
                                              target=PPConfig([(1, (1, edge)), (2, (edge + 1, 16))]))],
                    flags=flags or FeatureFlags())

    def fill(sim):
        store = sim.stores[2]
        for group in sorted(store.resident_groups):
            base = group * 1000
            store.append("zombie", group, ghost_tokens, [base + i for i in range(ghost_tokens)])

    return scen, fill


def fig3_cluster(mem_mib=4096):
    return {i: GpuSpec(id=i, mem_total=mem_mib * MIB, mem_bandwidth=1e12, prefill_cost=1e-6,
                       decode_cost=1e-5, alloc_granularity=2 * MIB) for i in (1, 2, 3)}


def fig3_model():
    return ModelSpec(num_layers=6, layer_weight_bytes=64 * MIB, token_kv_bytes_per_layer=8 * KIB,
                     stacking_factor=1, activation_bytes_per_token=2 * KIB)


def fig3_scenario(triggers=(), flags=None, num_requests=4, rate=200.0, pattern="decode_heavy",
                  tau=50) -> Scenario:
    return Scenario(cluster=list(fig3_cluster().values()), model=fig3_model(), initial_config=C_A,
                    workload=WorkloadSpec(pattern=pattern, rate=rate, num_requests=num_requests),
                    triggers=[ReconfigTrigger(at, tgt, tau=tau) for at, tgt in triggers],
                    flags=flags or FeatureFlags())


def golden_runs():
    """name -> (scenario, seed, fill) for every run recorded in tests/golden/simulations.json"""
    runs = {
        "fig3_seed5": (fig3_scenario(triggers=[(0.02, C_B)], num_requests=4, rate=500.0), 5, None),
        "hetero_c10_seed123": (hetero_scenario(rate=7.0, n=40), 123, None),
        "hetero_n60_seed7": (hetero_scenario(rate=7.0, n=60), 7, None),
        "fig3_nopatch": (fig3_scenario(triggers=[(0.02, C_B)], num_requests=4, rate=500.0,
                                       flags=FeatureFlags(kv_patch=False)), 5, None),
    }
    for L in (4, 8):
        scen, fill = stoptime_scenario(migrate_layers=L)
        runs[f"stoptime_L{L}"] = (scen, 0, fill)
    return runs
